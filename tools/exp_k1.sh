# Source-major K1 on C2: strip width x TMA element group at 2 stages; complex64 stages (bench)
export FWI_KKT_KM_STAGES=2
for cols in 64 32; do for g in 8 4 2; do
  FWI_KKT_KM_COLS=$cols FWI_KKT_GRP=$g timeout 120 python tools/apply_sizes.py c2
done; done
FWI_KKT_KM_COLS=32 FWI_KKT_KM_STAGES=3 timeout 120 python tools/apply_sizes.py c2
for s in 2 3 4; do
  FWI_KKT_KM_COLS=64 FWI_KKT_KM_STAGES=$s timeout 200 python bench.py --skip-cpu --skip-krylov --steps 300 | python -c "import json,sys; d=json.load(sys.stdin); print('bench cols64 S=$s', d['ms_per_step'], d['roofline']['frac'], d['c64'])"
done
