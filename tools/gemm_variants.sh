# A/B of K3 builds in build_variants/* (tools/mkvar_gemm.sh) with tools/gemm_probe.py
for v in "$@"; do echo "== $v"; WT_LIB_PATH=build_variants/$v/libwten_b200.so timeout 300 python tools/gemm_probe.py 2>&1 | grep -v "^cuBLAS" | head -12; done
