# usage: tools/mkvar_eig.sh name "defines" -> build_variants/lib_<name>.so (eig.cu rebuilt with the defines)
set -e
cd /root/repo/paper_2601_08228_b200/csrc
d=/root/repo/build_variants/$1; mkdir -p $d
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr $2 -c eig.cu -o $d/eig.o 2> $d/ptxas.log
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o /root/repo/build_variants/lib_$1.so build/wt_status.o build/lift.o build/lift_fast.o build/gemm.o build/svd.o $d/eig.o build/util.o build/epilogue.o build/wproduct.o build/imaging.o -lcudart
grep -A2 "sbr_update_mult" $d/ptxas.log | grep -i "registers\|spill" | tr '\n' ' '; echo " <- $1"
