# A/B of K4 builds in build_variants/* (tools/mkvar_svd.sh) on the config-3/4/5 SVD shapes.
for v in "$@"; do
  echo "== $v"
  for args in "256 192" "512 32" "1024 32"; do
    WT_LIB_PATH=build_variants/$v/libwten_b200.so timeout 120 python tools/svd_waves.py $args
  done
done
