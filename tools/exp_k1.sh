# Source-major K1 on C2: halo columns as separate boxes (hx, default) vs one widened box
timeout 120 python tools/apply_sizes.py c2
FWI_KKT_KM_HX=0 timeout 120 python tools/apply_sizes.py c2
FWI_KKT_KM_STAGES=3 timeout 120 python tools/apply_sizes.py c2
timeout 200 python bench.py --skip-cpu --skip-krylov --steps 300 | python -c "import json,sys; d=json.load(sys.stdin); print('bench', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), d['roofline']['kernel'][:40], round(d['c64']['frac'],3))"
