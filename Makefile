# Build recipe for the B200 energy-game solver and its test oracles.
#
#   make            product library paper_1710_03647_b200/libegs_b200.so (sm_100a)
#                   + oracle/libegs_oracle.so (C restatement, test-only)
#                   + oracle/_ref/libegsolve_ref.so when /root/reference exists
#   make clean
NVCC      ?= /usr/local/cuda/bin/nvcc
CXX       ?= g++
CC        ?= gcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v \
             --expt-relaxed-constexpr -Iinclude $(EXTRA_NVFLAGS)
PKG       := paper_1710_03647_b200
LIB       := $(PKG)/libegs_b200.so
CSRC      := $(PKG)/csrc
REF       ?= /root/reference/proj

ORACLE_LIB := oracle/libegs_oracle.so
ORACLE_CLI := oracle/egs_oracle_cli
REF_LIB    := oracle/_ref/libegsolve_ref.so

all: $(LIB) $(ORACLE_LIB) $(ORACLE_CLI) ref

HDRS := $(CSRC)/egs_types.cuh $(CSRC)/egs_device.cuh include/egs_gpu.h

$(CSRC)/egs_solver.o: $(CSRC)/egs_solver.cu $(CSRC)/egs_build.cuh $(CSRC)/egs_scan.cuh $(CSRC)/egs_narrow.h $(CSRC)/egs_pool.h $(HDRS)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(CSRC)/egs_solver.ptxas.log || (cat $(CSRC)/egs_solver.ptxas.log; false)
	sed -i '/Compile time/d' $(CSRC)/egs_solver.ptxas.log

# the solve kernels, once per edge-record format (8-byte int2 / packed 4-byte)
$(CSRC)/egs_kern_e8.o: $(CSRC)/egs_kern.cu $(CSRC)/egs_solve.cuh $(HDRS)
	$(NVCC) $(NVFLAGS) -DEGS_EDGE_BYTES=8 -DEGS_FMT_NS=e8 -c $< -o $@ 2> $(CSRC)/egs_kern_e8.ptxas.log || (cat $(CSRC)/egs_kern_e8.ptxas.log; false)
	sed -i '/Compile time/d' $(CSRC)/egs_kern_e8.ptxas.log

$(CSRC)/egs_kern_e4.o: $(CSRC)/egs_kern.cu $(CSRC)/egs_solve.cuh $(HDRS)
	$(NVCC) $(NVFLAGS) -DEGS_EDGE_BYTES=4 -DEGS_FMT_NS=e4 -c $< -o $@ 2> $(CSRC)/egs_kern_e4.ptxas.log || (cat $(CSRC)/egs_kern_e4.ptxas.log; false)
	sed -i '/Compile time/d' $(CSRC)/egs_kern_e4.ptxas.log

$(CSRC)/egs_host.o: $(CSRC)/egs_host.cpp $(CSRC)/egs_host_arena.h include/egs_gpu.h
	$(CXX) -O3 -std=c++17 -fPIC -Iinclude -I/usr/local/cuda/include -c $< -o $@

$(CSRC)/egs_arena_io.o: $(CSRC)/egs_arena_io.cpp $(CSRC)/egs_host_arena.h include/egs_gpu.h
	$(CXX) -O3 -std=c++17 -fPIC -Iinclude -c $< -o $@

$(CSRC)/egs_narrow.o: $(CSRC)/egs_narrow.cpp $(CSRC)/egs_narrow.h
	$(CXX) -O3 -std=c++17 -fPIC -c $< -o $@

$(LIB): $(CSRC)/egs_solver.o $(CSRC)/egs_kern_e8.o $(CSRC)/egs_kern_e4.o $(CSRC)/egs_host.o $(CSRC)/egs_arena_io.o $(CSRC)/egs_narrow.o
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $^ -lpthread

$(ORACLE_LIB): oracle/egs_oracle.c oracle/egs_oracle.h
	$(CC) -O2 -std=c11 -fPIC -shared -o $@ oracle/egs_oracle.c

$(ORACLE_CLI): oracle/egs_oracle_cli.c oracle/egs_oracle.c oracle/egs_oracle.h
	$(CC) -O2 -std=c11 -o $@ oracle/egs_oracle_cli.c oracle/egs_oracle.c

# The compiled reference (oracle/_ref): built from the reference sources where
# they lie, never copied.  `-include cmath` works around solver_seq.cpp:215
# calling llround without <cmath>.  Skipped when the reference is absent (the
# GPU box uses the prebuilt .so that travels with the snapshot).
ref: $(LIB)
	@if [ -d $(REF)/src ]; then $(MAKE) --no-print-directory $(REF_LIB) $(DROPIN_BINS); \
	 else echo "reference sources absent; using prebuilt $(REF_LIB) if present"; fi

REF_SRCS := $(wildcard $(REF)/src/*.cpp)
REF_OBJS := $(patsubst $(REF)/src/%.cpp,oracle/_ref/%.o,$(REF_SRCS))

oracle/_ref/%.o: $(REF)/src/%.cpp
	@mkdir -p oracle/_ref
	$(CXX) -std=c++20 -O3 -fPIC -include cmath -I$(REF)/include -c $< -o $@

oracle/_ref/ref_shim.o: oracle/ref_shim.cpp
	@mkdir -p oracle/_ref
	$(CXX) -std=c++20 -O3 -fPIC -I$(REF)/include -c $< -o $@

$(REF_LIB): $(REF_OBJS) oracle/_ref/ref_shim.o
	$(CXX) -shared -o $@ $^ -lpthread

# The C++ drop-in (integration/), compiled against the reference headers and
# linked with the reference library + libegs_b200.so: its parity test and
# the `egsolve solve` equivalent.  Built where /root/reference exists; the
# binaries travel to the GPU box with oracle/_ref.
DROPIN_BINS := oracle/_ref/test_solver_gpu oracle/_ref/egsolve_gpu
DROPIN_FLAGS := -std=c++20 -O2 -Iinclude -Iintegration -I$(REF)/include
DROPIN_LINK := oracle/_ref/solver_gpu.o -Loracle/_ref -legsolve_ref -L$(PKG) -l:libegs_b200.so \
	-Wl,-rpath,'$$ORIGIN:$$ORIGIN/../../$(PKG)' -lpthread

oracle/_ref/solver_gpu.o: integration/solver_gpu.cpp integration/solver_gpu.hpp include/egs_gpu.h
	@mkdir -p oracle/_ref
	$(CXX) $(DROPIN_FLAGS) -fPIC -c $< -o $@

oracle/_ref/test_solver_gpu: tests/cpp/test_solver_gpu.cpp oracle/_ref/solver_gpu.o $(REF_LIB) $(LIB)
	$(CXX) $(DROPIN_FLAGS) $< -o $@ $(DROPIN_LINK)

oracle/_ref/egsolve_gpu: integration/egsolve_gpu.cpp oracle/_ref/solver_gpu.o $(REF_LIB) $(LIB)
	$(CXX) $(DROPIN_FLAGS) $< -o $@ $(DROPIN_LINK)

clean:
	rm -f $(CSRC)/*.o $(LIB) $(ORACLE_LIB) $(ORACLE_CLI) oracle/_ref/*.o $(REF_LIB) $(DROPIN_BINS)

.PHONY: all ref clean
