# source-major K1: 1024 threads with one row per thread against 512 threads with two
# (config 2, both precisions, 2 and 3 stages)
export FWI_KKT_KM_LOG=1
for i in 1 2; do
python tools/apply_sizes.py c2
FWI_KKT_KM_THR=1024 python tools/apply_sizes.py c2
python tools/apply_sizes.py c2 c64
FWI_KKT_KM_THR=1024 python tools/apply_sizes.py c2 c64
FWI_KKT_KM_THR=1024 FWI_KKT_KM_STAGES=3 python tools/apply_sizes.py c2 c64
FWI_KKT_KM_THR=1024 FWI_KKT_KM_KS=1 FWI_KKT_KM_STAGES=3 python tools/apply_sizes.py c2 c64
done
