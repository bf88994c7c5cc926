# source-major K1 ring disciplines on config 2: block barrier (WS=0) vs per-stage empty barriers
# (WS=2), stages, and complex64 with two sources per stage (KS=2)
for v in "" "FWI_KKT_KM_WS=2 FWI_KKT_KM_STAGES=2" "FWI_KKT_KM_WS=2 FWI_KKT_KM_STAGES=3" "FWI_KKT_KM_WS=2 FWI_KKT_KM_STAGES=4" "FWI_KKT_KM_STAGES=3"; do
  env $v timeout 120 python tools/apply_sizes.py c2
done
for v in "" "FWI_KKT_KM_KS=2 FWI_KKT_KM_STAGES=2" "FWI_KKT_KM_KS=2 FWI_KKT_KM_STAGES=3" "FWI_KKT_KM_WS=2 FWI_KKT_KM_STAGES=3" "FWI_KKT_KM_WS=2 FWI_KKT_KM_STAGES=4" "FWI_KKT_KM_WS=2 FWI_KKT_KM_KS=2 FWI_KKT_KM_STAGES=2" "FWI_KKT_KM_WS=2 FWI_KKT_KM_KS=2 FWI_KKT_KM_STAGES=3" "FWI_KKT_KM_WS=2 FWI_KKT_KM_KS=2 FWI_KKT_KM_STAGES=4"; do
  env $v timeout 120 python tools/apply_sizes.py c2 c64
done
