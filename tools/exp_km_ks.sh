# complex128 source-major K1 with two sources per stage (half the steps and barriers, 88 KB stages)
for i in 1 2; do
python tools/apply_sizes.py c2
FWI_KKT_KM_KS=2 python tools/apply_sizes.py c2
FWI_KKT_KM_KS=2 FWI_KKT_KM_WS=2 FWI_KKT_KM_STAGES=2 python tools/apply_sizes.py c2
done
