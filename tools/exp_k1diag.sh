# K1 (tile TMA) on C2: full, data movement only, no stores, reads only; C3; C2 c64 via bench
timeout 120 python tools/apply_sizes.py c2
FWI_KKT_MEMONLY=1 timeout 120 python tools/apply_sizes.py c2
FWI_KKT_MEMONLY=1 FWI_KKT_NOSTORE=1 timeout 120 python tools/apply_sizes.py c2
FWI_KKT_MEMONLY=1 FWI_KKT_NOSTORE=1 FWI_KKT_NOFOLD=2 timeout 120 python tools/apply_sizes.py c2
timeout 120 python tools/apply_sizes.py c3
timeout 200 python bench.py --skip-cpu --skip-krylov --steps 300 | python -c "import json,sys; d=json.load(sys.stdin); print('bench', d['ms_per_step'], d['roofline']['frac'], d['c64'])"
