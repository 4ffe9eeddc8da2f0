# Build the sm_100a step library and the CPU oracle (test infrastructure).
#   make            -> paper_2509_04277_b200/librodsim_b200.so, oracle/liboracle.so
#   make ref        -> oracle/_ref (the reference's own compiled core, if present)
NVCC    ?= nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -std=c++17 $(ARCH) -O3 -lineinfo -Xcompiler -fPIC -Xptxas -v
CSRC    := paper_2509_04277_b200/csrc
LIB     := paper_2509_04277_b200/librodsim_b200.so
HDRS    := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.h) include/rodsim_b200.h
OBJS    := build/rod_kernels_mirror.o build/rod_kernels_fast.o build/rodsim_capi.o build/rod_micro.o

all: $(LIB) oracle/liboracle.so

build:
	mkdir -p build

# fp64 mirror: no FMA contraction, IEEE division and square root
build/rod_kernels_mirror.o: $(CSRC)/rod_kernels_mirror.cu $(HDRS) | build
	$(NVCC) $(NVFLAGS) --fmad=false -prec-div=true -prec-sqrt=true -c $< -o $@ 2> build/ptxas_mirror.log || (cat build/ptxas_mirror.log; false)

build/rod_kernels_fast.o: $(CSRC)/rod_kernels_fast.cu $(HDRS) | build
	$(NVCC) $(NVFLAGS) --fmad=true -c $< -o $@ 2> build/ptxas_fast.log || (cat build/ptxas_fast.log; false)

# latency microbenchmarks, mirror flags (the chains the mirror kernel issues)
build/rod_micro.o: $(CSRC)/rod_micro.cu $(CSRC)/rod_math.cuh | build
	$(NVCC) -std=c++17 $(ARCH) -O3 -lineinfo -Xcompiler -fPIC --fmad=false -prec-div=true -prec-sqrt=true -c $< -o $@

build/rodsim_capi.o: $(CSRC)/rodsim_capi.cu $(HDRS) | build
	$(NVCC) -std=c++17 $(ARCH) -O2 -Xcompiler -fPIC -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared $(OBJS) -o $@

# CPU restatement of the reference step (tests/bench checker only)
oracle/liboracle.so: oracle/rod_oracle.c oracle/rod_oracle.h
	gcc -O2 -fPIC -ffp-contract=off -fno-math-errno -shared $< -o $@ -lm

ref:
	./oracle/build_ref.sh

clean:
	rm -rf build $(LIB) oracle/liboracle.so

.PHONY: all ref clean
