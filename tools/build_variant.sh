# Build an alternative libegs_b200.so with extra kernel defines into
# scratch_libs/<name>/ (tuning experiments; select with EGS_LIB=...).
#   bash tools/build_variant.sh <name> -DEGS_FOO=1 ...
set -eu
name=$1; shift
out=scratch_libs/$name
mkdir -p $out
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude $*"
C=paper_1710_03647_b200/csrc
$NV -DEGS_EDGE_BYTES=8 -DEGS_FMT_NS=e8 -c $C/egs_kern.cu -o $out/e8.o &
$NV -DEGS_EDGE_BYTES=4 -DEGS_FMT_NS=e4 -c $C/egs_kern.cu -o $out/e4.o &
$NV -c $C/egs_solver.cu -o $out/solver.o &  # (host constants may follow the defines)
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $out/libegs_b200.so $out/solver.o $out/e8.o $out/e4.o $C/egs_host.o $C/egs_arena_io.o $C/egs_narrow.o -lpthread
echo $out/libegs_b200.so
