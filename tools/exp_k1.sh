# Source-major K1: complex64 sources per stage x ring depth (bench c64 line); complex128 default
for sps in 2 1; do for st in 2 3; do
  FWI_KKT_KM_SPS=$sps FWI_KKT_KM_STAGES=$st timeout 200 python bench.py --skip-cpu --skip-krylov --steps 300 | python -c "import json,sys; d=json.load(sys.stdin); print('sps=$sps S=$st', round(d['ms_per_step'],4), round(d['roofline']['frac'],3), round(d['c64']['ms_per_apply'],4), round(d['c64']['frac'],3), d['c64']['kernel'][:40])"
done; done
