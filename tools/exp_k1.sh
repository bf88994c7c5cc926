# Chunked tile kernel with L1::no_allocate stores: C2 (forced), C3, C5
FWI_KKT_KERNEL=tile timeout 120 python tools/apply_sizes.py c2
timeout 120 python tools/apply_sizes.py c3
timeout 600 python tools/c5_apply.py 20 2>&1 | tail -2
