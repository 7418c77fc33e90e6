# Round-2 evidence refresh on one B200: GPU tests, smoke, bench (ours + reference arm, the
# driver's flags), the ncu launch list of the bench, ncu --set full captures of the K4
# kernels on configs 3 / 4 (Jacobi sweep, tridiagonalization panel), K3 and K1/K2.
set -x
mkdir -p gpurun_out/r02
O=gpurun_out/r02
timeout 1200 python -m pytest tests -m gpu -q > $O/gputests.log 2>&1; echo rc=$? >> $O/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2000 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --workloads none --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:svd_sweep_kernel --launch-skip 2 -c 1 -o $O/k4_sweep_cfg4 -f python tools/eig_one.py 4 > $O/ncu_k4_4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tridiag_panel --launch-skip 40 -c 1 -o $O/k4_tridiag_cfg4 -f python tools/eig_one.py 4 > $O/ncu_tri4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:svd_sweep_kernel --launch-skip 2 -c 1 -o $O/k4_sweep_cfg3 -f python tools/eig_one.py 3 > $O/ncu_k4_3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_f64_kernel -c 1 -o $O/gemm -f python tools/gemm_one.py > $O/ncu_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"fwd_|inv_" -c 8 -o $O/lift -f python tools/lift_one.py 1 2 4 8 > $O/ncu_lift.log 2>&1
