# source-major K1 with balanced rectangles (one per CTA) on configs 2 and 3, both precisions,
# against equal strips and the chunked tile kernel
export FWI_KKT_KM_LOG=1
python tools/apply_sizes.py c2
FWI_KKT_KM_BALANCED=1 python tools/apply_sizes.py c2
python tools/apply_sizes.py c2 c64

FWI_KKT_KM_BALANCED=1 python tools/apply_sizes.py c3
FWI_KKT_KM_BALANCED=1 python tools/apply_sizes.py c3 c64
FWI_KKT_KERNEL=tile python tools/apply_sizes.py c3
FWI_KKT_KERNEL=tile python tools/apply_sizes.py c3 c64
