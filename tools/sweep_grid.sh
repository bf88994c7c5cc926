# per-step time of the exact sweep (config 1, 8 RHS) per launch shape and line orientation
for o in short long; do for v in "16 1 1" "16 2 1" "16 4 1" "16 8 1" "16 4 2" "16 8 2" "8 2 1" "8 8 1"; do
  set -- $v
  echo -n "$o CS=$1 KG=$2 KR=$3: "
  FWI_EXACT_LINES=$o FWI_EXACT_CS=$1 FWI_EXACT_KG=$2 FWI_EXACT_KR=$3 python tools/sweep_trace.py c1 2>&1 | grep "per-step" | awk '{print $5, $6, $7, $8}'
done; done
