# precond_apply device time on config 3 (2 x 48-RHS exact solves) per sweep launch shape
for v in "16 8 2" "16 8 1" "16 6 1" "16 4 1" "8 8 1" "8 8 2"; do
  set -- $v
  echo -n "CS=$1 KG=$2 KR=$3: "
  FWI_EXACT_CS=$1 FWI_EXACT_KG=$2 FWI_EXACT_KR=$3 python tools/krylov_parts.py c3 2>&1 | grep precond_apply
done
echo -n "auto: "; python tools/krylov_parts.py c3 2>&1 | grep -E "precond_apply|fsgn" | tail -2
