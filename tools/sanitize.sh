# compute-sanitizer over tools/sanitize_cases.py (small sizes)
out=gpurun_out/sanitizer
mkdir -p $out
CS="compute-sanitizer --print-limit 20 --error-exitcode 9"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 $CS --tool $tool python tools/sanitize_cases.py all > $out/$tool.log 2>&1; echo "$tool rc=$?" >> $out/summary.txt
done
for S in 2 4 8; do
  WT_OPT_SVD_SPLIT=$S timeout 900 $CS --tool memcheck python tools/sanitize_cases.py svd > $out/memcheck_split$S.log 2>&1; echo "memcheck split $S rc=$?" >> $out/summary.txt
  WT_OPT_SVD_SPLIT=$S timeout 900 $CS --tool racecheck python tools/sanitize_cases.py svd > $out/racecheck_split$S.log 2>&1; echo "racecheck split $S rc=$?" >> $out/summary.txt
done
WT_OPT_SVD_PRECOND=0 timeout 900 $CS --tool racecheck python tools/sanitize_cases.py svd > $out/racecheck_noprecond.log 2>&1; echo "racecheck no-precond rc=$?" >> $out/summary.txt
cat $out/summary.txt
