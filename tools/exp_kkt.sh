run() { env "$@" python bench.py --skip-cpu --skip-krylov 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$*', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), round(d['c64']['ms_per_apply'],4), round(d['c64']['frac'],3))"; }
run X=tma
run FWI_KKT_LOADER=cpasync
run FWI_KKT_LOADER=cpasync FWI_KKT_STAGES=2
run FWI_KKT_LOADER=cpasync FWI_KKT_MEMONLY=1 FWI_KKT_NOSTORE=1 FWI_KKT_NOFOLD=1
FWI_KKT_LOADER=cpasync python -m pytest tests/test_gpu_parity.py -q -m gpu -k "kkt_apply or c64" 2>&1 | tail -1
