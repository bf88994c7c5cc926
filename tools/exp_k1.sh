# Source-major K1 (equal runs per SM) on C2 for strip widths 64/32/128; C3; complex64 via bench
for cols in 64 32 128; do FWI_KKT_KM_COLS=$cols timeout 120 python tools/apply_sizes.py c2; done
FWI_KKT_KM_STAGES=3 timeout 120 python tools/apply_sizes.py c2
timeout 120 python tools/apply_sizes.py c3
FWI_KKT_KM_FORCE=1 timeout 120 python tools/apply_sizes.py c3
timeout 200 python bench.py --skip-cpu --skip-krylov --steps 300 | python -c "import json,sys; d=json.load(sys.stdin); print('bench', d['ms_per_step'], d['roofline']['frac'], d['c64'])"
