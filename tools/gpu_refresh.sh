# Round-2 evidence refresh on one B200: GPU tests, smoke, bench (ours + reference arm, the
# driver's flags), the ncu launch list of the bench, per-phase launch lists of one K4 call
# (configs 3, 4 full, 4 leading-triplet), ncu --set full captures of the K4 kernels (Jacobi
# sweep, one-stage tridiagonalization panel on config 3, the two-stage trailing pass / band
# chase / panel QR on config 4), K3 and K1/K2.
set -x
mkdir -p gpurun_out/r02
O=gpurun_out/r02
timeout 1200 python -m pytest tests -m gpu -q > $O/gputests.log 2>&1; echo rc=$? >> $O/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.json 2> $O/bench_ref.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -c 2000 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --workloads none --no-cpu-baseline > $O/ncu_launch.log 2>&1
for c in 4t 4 3; do
  timeout 600 ncu --nvtx --nvtx-include "k4call/" --metrics $M --clock-control none --csv --log-file $O/k4_$c.csv python tools/k4_launches.py $c > $O/k4_$c.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:svd_sweep_kernel --launch-skip 2 -c 1 -o $O/k4_sweep_cfg4 -f python tools/eig_one.py 4 > $O/ncu_k4_4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sbr_update_mult --launch-skip 88 -c 1 -o $O/k4_trailing_cfg4 -f python tools/sbr_probe.py 32 > $O/ncu_um.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sbr_chase --launch-skip 1 -c 1 -o $O/k4_chase_cfg4 -f python tools/sbr_probe.py 32 > $O/ncu_chase.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sbr_panel --launch-skip 96 -c 1 -o $O/k4_panelqr_cfg4 -f python tools/sbr_probe.py 32 > $O/ncu_pqr.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tridiag_panel --launch-skip 4 -c 1 -o $O/k4_tridiag_cfg3 -f python tools/eig_one.py 3 > $O/ncu_tri3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:svd_sweep_kernel --launch-skip 2 -c 1 -o $O/k4_sweep_cfg3 -f python tools/eig_one.py 3 > $O/ncu_k4_3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_f64_kernel -c 1 -o $O/gemm -f python tools/gemm_one.py > $O/ncu_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"fwd_|inv_" -c 8 -o $O/lift -f python tools/lift_one.py 1 2 4 8 > $O/ncu_lift.log 2>&1
timeout 600 ncu --metrics $M --clock-control none -c 200 --csv --log-file $O/imaging_launches.csv python tools/imaging_probe.py > $O/ncu_imaging.log 2>&1
timeout 900 python tools/fuzz_parity.py 200 7 > $O/fuzz.log 2>&1
for f in $O/*.ncu-rep; do ncu -i $f --page raw --csv > ${f%.ncu-rep}_raw.csv 2>/dev/null; done
