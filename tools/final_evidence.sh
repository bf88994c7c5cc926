# Round-2 evidence capture on one B200 (outputs under gpurun_out/ev/): smoke, the GPU suite, the
# bench line, the bench's launch list, ncu captures of the production K1 (c128 and c64), the
# C1/C3 Krylov kernel splits and one C3 exact precond_apply's launch list
set -x
mkdir -p gpurun_out/ev
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/ev/gputest.log 2>&1
python bench.py > gpurun_out/ev/bench.json 2> gpurun_out/ev/bench.err
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/ev/bench_ref.json 2> gpurun_out/ev/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev/launches_bench.csv \
    python bench.py --steps 20 --warmup 3 --skip-cpu --skip-krylov > gpurun_out/ev/ncu_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:kkt_km1 -s 2 -c 1 -o gpurun_out/ev/km1_c128 \
    python tools/prof_kkt.py --what apply > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:kkt_km1 -s 2 -c 1 -o gpurun_out/ev/km1_c64 \
    python tools/prof_kkt.py --what apply32 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --profile-from-start off --csv \
    --log-file gpurun_out/ev/krylov_c1.csv python tools/krylov_prof.py c1 > gpurun_out/ev/krylov_c1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --profile-from-start off --csv \
    --log-file gpurun_out/ev/krylov_c3.csv python tools/krylov_prof.py c3 > gpurun_out/ev/krylov_c3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/ev/bcr_c3.csv python tools/bcr_prof.py > /dev/null 2>&1
python tools/krylov_ab.py all > gpurun_out/ev/krylov_ab.log 2>&1
python tools/k1_timeline.py c128 gpurun_out/ev/k1_timeline_c128.json > gpurun_out/ev/k1_timeline_c128.log 2>&1
python tools/k1_timeline.py c64 gpurun_out/ev/k1_timeline_c64.json > gpurun_out/ev/k1_timeline_c64.log 2>&1
FWI_KKT_KM_RDUP=1 python tools/apply_sizes.py c2 > gpurun_out/ev/k1_rdup_ab.log 2>&1
python tools/apply_sizes.py c2 >> gpurun_out/ev/k1_rdup_ab.log 2>&1
FWI_KKT_KM_RDUP=1 python tools/apply_sizes.py c2 c64 >> gpurun_out/ev/k1_rdup_ab.log 2>&1
python tools/apply_sizes.py c2 c64 >> gpurun_out/ev/k1_rdup_ab.log 2>&1
