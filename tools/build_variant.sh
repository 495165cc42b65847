# build an experimental copy of the library with extra -D flags:
#   bash tools/build_variant.sh <name> -DFOO ...  -> build/var_<name>/libdgc_b200.so
name=$1; shift
d=build/var_$name; mkdir -p $d
ARCH="-gencode arch=compute_100a,code=sm_100a"
for f in common spmm stale exchange dense rnn gemm_tc rnn_tc evolve; do
  nvcc $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC "$@" -c paper_2309_03523_b200/csrc/$f.cu -o $d/$f.o &
done
wait
nvcc $ARCH -shared --cudart static -o $d/libdgc_b200.so $d/*.o build/layout.o build/fusion_plan.o
