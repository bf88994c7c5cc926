# Source-major K1 on C2: u via registers (default) vs a third TMA box; ring depth
timeout 120 python tools/apply_sizes.py c2
FWI_KKT_KM_ULDG=0 timeout 120 python tools/apply_sizes.py c2
FWI_KKT_KM_STAGES=3 timeout 120 python tools/apply_sizes.py c2
FWI_KKT_GRP=4 timeout 120 python tools/apply_sizes.py c2
timeout 200 python bench.py --skip-cpu --skip-krylov --steps 300 | python -c "import json,sys; d=json.load(sys.stdin); print('bench', d['ms_per_step'], d['roofline']['frac'], d['c64'])"
FWI_KKT_KM_STAGES=2 timeout 200 python bench.py --skip-cpu --skip-krylov --steps 300 | python -c "import json,sys; d=json.load(sys.stdin); print('bench c64 S=2', d['c64'])"
