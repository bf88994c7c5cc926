run() { env "$@" python bench.py --skip-cpu --skip-krylov 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$*', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), round(d['c64']['ms_per_apply'],4), round(d['c64']['frac'],3))"; }
run X=512x128
cp paper_2204_06489_b200/libfwi_b200.so /tmp/keep.so
for v in 256_64 256_128; do cp tools/lib_$v.so paper_2204_06489_b200/libfwi_b200.so; run X=$v; run X=$v FWI_KKT_STAGES=2; done
cp tools/lib_256_64.so paper_2204_06489_b200/libfwi_b200.so; python -m pytest tests/test_gpu_parity.py -q -m gpu -k "kkt_apply or c64" 2>&1 | tail -1
cp /tmp/keep.so paper_2204_06489_b200/libfwi_b200.so
