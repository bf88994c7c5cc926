# config 3: source-major K1 with taller bands (fewer CTAs) against the chunked tile kernel
timeout 120 python tools/apply_sizes.py c3
for r in 6 8 11 16; do FWI_KKT_KM_FORCE=1 FWI_KKT_KM_ROWS=$r timeout 120 python tools/apply_sizes.py c3; done
FWI_KKT_KM_FORCE=1 FWI_KKT_KM_ROWS=11 FWI_KKT_KM_STAGES=3 timeout 120 python tools/apply_sizes.py c3
