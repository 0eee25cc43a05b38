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

$(CSRC)/egs_solver.o: $(CSRC)/egs_solver.cu $(CSRC)/egs_solve.cuh $(CSRC)/egs_build.cuh $(CSRC)/egs_device.cuh include/egs_gpu.h
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(CSRC)/egs_solver.ptxas.log || (cat $(CSRC)/egs_solver.ptxas.log; false)

$(CSRC)/egs_host.o: $(CSRC)/egs_host.cpp include/egs_gpu.h
	$(CXX) -O3 -std=c++17 -fPIC -Iinclude -I/usr/local/cuda/include -c $< -o $@

$(LIB): $(CSRC)/egs_solver.o $(CSRC)/egs_host.o
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $^ -lpthread

$(ORACLE_LIB): oracle/egs_oracle.c oracle/egs_oracle.h
	$(CC) -O2 -std=c11 -fPIC -shared -o $@ oracle/egs_oracle.c

$(ORACLE_CLI): oracle/egs_oracle_cli.c oracle/egs_oracle.c oracle/egs_oracle.h
	$(CC) -O2 -std=c11 -o $@ oracle/egs_oracle_cli.c oracle/egs_oracle.c

# The compiled reference (oracle/_ref): built from the reference sources where
# they lie, never copied.  `-include cmath` works around solver_seq.cpp:215
# calling llround without <cmath>.  Skipped when the reference is absent (the
# GPU box uses the prebuilt .so that travels with the snapshot).
ref:
	@if [ -d $(REF)/src ]; then $(MAKE) --no-print-directory $(REF_LIB); \
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

clean:
	rm -f $(CSRC)/*.o $(LIB) $(ORACLE_LIB) $(ORACLE_CLI) oracle/_ref/*.o $(REF_LIB)

.PHONY: all ref clean
