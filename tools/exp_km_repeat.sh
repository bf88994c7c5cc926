for i in 1 2 3; do
python tools/apply_sizes.py c2
python tools/apply_sizes.py c2 c64
done
