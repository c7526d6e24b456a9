# Round evidence on one B200 (run through gpurun from the repo root): GPU tests, bench lines,
# launch list and ncu captures of the dominant kernels.  Outputs land in gpurun_out/.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/gputests.log
timeout 300 python bench.py > gpurun_out/bench_default.log 2>&1
timeout 300 python bench.py --dim 3 --degree 3 --no-cpu > gpurun_out/bench_3d.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_k4.csv python bench.py --steps 3 --warmup 3 --no-pcg --no-cpu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"apply2d|patch_fdm2d_mma" -c 2 -o gpurun_out/rx_2d_k4_avs python tools/prof_step.py --degree 4 --sm avs_atomic --reps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"mvs2d_mma" -c 1 -o gpurun_out/rx_2d_k4_mvs python tools/prof_step.py --degree 4 --sm mvs --reps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"apply3d|patch_fdm3d" -c 2 -o gpurun_out/rx_3d_k3_avs python tools/prof_step.py --dim 3 --degree 3 --sm avs_atomic --reps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"mvs3d" -c 1 -o gpurun_out/rx_3d_k3_mvs python tools/prof_step.py --dim 3 --degree 3 --sm mvs --reps 1 > /dev/null 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
cat gpurun_out/gputests.log gpurun_out/smoke.log
