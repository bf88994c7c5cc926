run() { env "$@" python bench.py --skip-cpu --skip-krylov 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$*', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), round(d['c64']['ms_per_apply'],4), round(d['c64']['frac'],3))"; }
run FWI_KKT_STAGES=2
run FWI_KKT_STAGES=4
run FWI_KKT_F32_TMA=1
