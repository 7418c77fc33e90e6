# A/B of eig.cu build variants (build_variants/lib_*.so) on the precond check
for lib in paper_2601_08228_b200/libwten_b200.so build_variants/lib_*.so; do
  echo "== $lib"
  WT_LIB_PATH=$PWD/$lib WT_OPT_EIG_PROFILE=1 timeout 300 python tools/precond_check.py 2>&1 | grep -E "cfg3|cfg4|wt_eig\] n=(256 batch=192|1024 batch=32)" | awk '!seen[$0]++' | tail -4
done
