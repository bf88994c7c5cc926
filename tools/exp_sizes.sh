for c in c3 c2; do
python tools/apply_sizes.py $c
FWI_KKT_KERNEL=plain python tools/apply_sizes.py $c
FWI_KKT_KC=4 python tools/apply_sizes.py $c
FWI_KKT_KC=8 python tools/apply_sizes.py $c
FWI_KKT_KC=1 python tools/apply_sizes.py $c
done
