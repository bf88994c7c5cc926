# K1 variants on C2 (ms per apply, HBM fraction) via the plan's env knobs
run() { env "$@" timeout 120 python bench.py --skip-cpu --skip-krylov --steps 300 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$*', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), round(d['c64']['ms_per_apply'],4), round(d['c64']['frac'],3))"; }
run X=default
run FWI_KKT_WS=2
run X=default
run FWI_KKT_WS=2
for c in c3 c2; do timeout 120 python tools/apply_sizes.py $c; FWI_KKT_WS=2 timeout 120 python tools/apply_sizes.py $c; done
