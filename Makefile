# Build the sm_100a step library and the CPU oracle (test infrastructure).
#   make            -> paper_2509_04277_b200/librodsim_b200.so, oracle/liboracle.so
#   make ref        -> oracle/_ref (the reference's own compiled core, if present)
NVCC    ?= nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
# PROF=1 compiles in the per-phase cycle profile (RSB_DEBUG=2 at run time;
# rebuild from clean when toggling)
PROF    ?= 0
NVFLAGS := -std=c++17 $(ARCH) -O3 -lineinfo -Xcompiler -fPIC -Xptxas -v -DRSB_PROF=$(PROF)
CSRC    := paper_2509_04277_b200/csrc
LIB     := paper_2509_04277_b200/librodsim_b200.so
HDRS    := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.h) include/rodsim_b200.h
KOBJS   := build/k_mirror.o build/k_mirror_feat.o build/k_f32.o build/k_f32_feat.o \
           build/k_f64fast.o build/k_f64fast_feat.o
OBJS    := $(KOBJS) build/rodsim_capi.o build/rod_micro.o
MIRROR  := --fmad=false -prec-div=true -prec-sqrt=true
FAST    := --fmad=true
KSRC    := $(CSRC)/rod_kernels.cu

all: $(LIB) oracle/liboracle.so

build:
	mkdir -p build

# the step kernel: one object per precision mode x scene features, built in
# parallel (csrc/rod_kernels.cu).  mirror = fp64 with the reference's
# rounding (no FMA contraction, IEEE division and square root).
build/k_%.o: $(KSRC) $(HDRS) | build
	$(NVCC) $(NVFLAGS) $(KFLAGS_$*) -c $< -o $@ 2> build/ptxas_$*.log || (cat build/ptxas_$*.log; false)

KFLAGS_mirror       := $(MIRROR) -DRSB_MODE_NS=mirror -DRSB_MODE_ID=0 -DRSB_REAL=double -DRSB_FEAT=0
KFLAGS_mirror_feat  := $(MIRROR) -DRSB_MODE_NS=mirror_feat -DRSB_MODE_ID=0 -DRSB_REAL=double -DRSB_FEAT=1
KFLAGS_f32          := $(FAST) -DRSB_MODE_NS=f32 -DRSB_MODE_ID=1 -DRSB_REAL=float -DRSB_FEAT=0
KFLAGS_f32_feat     := $(FAST) -DRSB_MODE_NS=f32_feat -DRSB_MODE_ID=1 -DRSB_REAL=float -DRSB_FEAT=1
KFLAGS_f64fast      := $(FAST) -DRSB_MODE_NS=f64fast -DRSB_MODE_ID=1 -DRSB_REAL=double -DRSB_FEAT=0
KFLAGS_f64fast_feat := $(FAST) -DRSB_MODE_NS=f64fast_feat -DRSB_MODE_ID=1 -DRSB_REAL=double -DRSB_FEAT=1

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
