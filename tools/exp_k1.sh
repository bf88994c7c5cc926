timeout 120 python tools/apply_sizes.py c2
timeout 600 python tools/c5_apply.py 20 2>&1 | tail -1
