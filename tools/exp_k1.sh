# Source-major K1 forced on C3 (bands < 8 rows) against the chunked tile kernel
timeout 120 python tools/apply_sizes.py c3
for cols in 128 64 32; do FWI_KKT_KM_FORCE=1 FWI_KKT_KM_COLS=$cols timeout 120 python tools/apply_sizes.py c3; done
