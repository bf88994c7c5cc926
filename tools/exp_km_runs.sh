# (record of a removed experiment: the row-run kernel variant (FWI_KKT_KM_CROSS, FWI_KKT_KM_X2RECT)
# was measured slower and not committed, profiles/r02_k1_row_runs.log)
# source-major K1: row runs crossing strip ends (X2, 148 CTAs of 13-14 rows on config 2) against
# one rectangle per CTA (144 CTAs of 14-15 rows); FWI_KKT_KM_X2RECT=1 runs the X2 kernel on the
# rectangles (separates the kernel's cost from the layout's)
export FWI_KKT_KM_LOG=1
for i in 1 2; do
python tools/apply_sizes.py c2
FWI_KKT_KM_CROSS=0 python tools/apply_sizes.py c2
FWI_KKT_KM_CROSS=0 FWI_KKT_KM_X2RECT=1 python tools/apply_sizes.py c2
python tools/apply_sizes.py c2 c64
FWI_KKT_KM_CROSS=0 python tools/apply_sizes.py c2 c64
FWI_KKT_KM_CROSS=0 FWI_KKT_KM_X2RECT=1 python tools/apply_sizes.py c2 c64
done
