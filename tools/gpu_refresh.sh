# Round-end evidence refresh on one B200: GPU tests, bench (ours + reference arm),
# ncu launch list of the bench, ncu --set full captures of the K4 sweep kernel
# (configs 3 and 4), the K3 face GEMM and the config-2 lifting launches.
set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo rc=$? >> gpurun_out/gputests.log
timeout 400 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 400 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:svd_sweep_kernel --launch-skip 6 -c 1 -o gpurun_out/k4_cfg3 -f python tools/svd_one.py 3 > gpurun_out/ncu_k4_3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:svd_sweep_kernel --launch-skip 6 -c 1 -o gpurun_out/k4_cfg4 -f python tools/svd_one.py 4 > gpurun_out/ncu_k4_4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_f64_kernel -c 1 -o gpurun_out/gemm -f python tools/gemm_one.py > gpurun_out/ncu_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"fwd_|inv_" -c 8 -o gpurun_out/lift -f python tools/lift_one.py 1 2 4 8 > gpurun_out/ncu_lift.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:svd_sweep_kernel --launch-skip 6 -c 1 -o gpurun_out/k4_split -f python tools/svd_split_one.py > gpurun_out/ncu_k4_split.log 2>&1
