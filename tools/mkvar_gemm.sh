# usage: mkgemm.sh name "defines"  -> build_variants/<name>/libwten_b200.so with a gemm.cu variant
set -e
cd /root/repo/paper_2601_08228_b200/csrc
d=/root/repo/build_variants/$1; mkdir -p $d
nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr $2 -c gemm.cu -o $d/gemm.o 2> $d/ptxas.log
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $d/libwten_b200.so build/wt_status.o build/lift.o build/lift_fast.o $d/gemm.o build/svd.o build/util.o build/epilogue.o -lcudart
grep -A2 "gemm_f64_kernelILi128ELi128ELi2ELi4ELb0ELb0ELi2" $d/ptxas.log | grep -i "registers\|spill" | tr '\n' ' '; echo " <- $1"
