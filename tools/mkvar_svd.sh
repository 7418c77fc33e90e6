# usage: mkvar.sh name "defines"
set -e
cd /root/repo/paper_2601_08228_b200/csrc
d=/root/repo/build_variants/$1; mkdir -p $d
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr $2 -c svd.cu -o $d/svd.o 2> $d/ptxas.log
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/libwten_b200.so build/wt_status.o build/lift.o build/lift_fast.o build/gemm.o $d/svd.o build/util.o build/epilogue.o -lcudart
grep -A2 "sweep_kernel" $d/ptxas.log | grep -i "registers\|spill" | tr '\n' ' '; echo " <- $1"
