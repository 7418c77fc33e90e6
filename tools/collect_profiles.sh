# gpurun_out/r02 (tools/gpu_refresh.sh) -> profiles/ (tracked evidence of round 2)
set -e
O=gpurun_out/r02
cp $O/bench.json profiles/r02_bench.json
cp $O/bench_ref.json profiles/r02_bench_reference.json
cp $O/launches.csv profiles/r02_bench_launches.csv
python tools/ncu_summary.py $O/*.ncu-rep > profiles/r02_ncu_kernels.jsonl
rm -f profiles/traffic_r02.json
for c in 4t 4 3; do python tools/k4_traffic.py $O/k4_$c.csv $c profiles/traffic_r02.json > /dev/null; done
for k in k4_trailing_cfg4 k4_chase_cfg4 k4_panelqr_cfg4 k4_tridiag_cfg3; do
  python tools/ncu_lines.py $O/$k.ncu-rep 14 > profiles/r02_lines_$k.txt
done
python tools/launch_summary.py $O/imaging_launches.csv > profiles/r02_imaging_launches.txt
tail -1 $O/fuzz.log > profiles/r02_fuzz_tail.txt
tail -3 $O/gputests.log > profiles/r02_gputests_tail.txt
tail -2 $O/smoke.log >> profiles/r02_gputests_tail.txt
