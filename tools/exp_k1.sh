# Source-major K1 on C2 with L1::no_allocate stores: ring depth, unused smem, c64
export FWI_KKT_KM_ST=1
for s in 2 3 4; do FWI_KKT_KM_STAGES=$s timeout 120 python tools/apply_sizes.py c2; done
FWI_KKT_KM_PAD_KB=60 timeout 120 python tools/apply_sizes.py c2
FWI_KKT_KM_ULDG=0 timeout 120 python tools/apply_sizes.py c2
for s in 2 3 4; do FWI_KKT_KM_STAGES=$s timeout 200 python bench.py --skip-cpu --skip-krylov --steps 300 | python -c "import json,sys; d=json.load(sys.stdin); print('bench S=$s', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), round(d['c64']['ms_per_apply'],4), round(d['c64']['frac'],3))"; done
