# Build libttc.so (product, sm_100a) and liboracle.so (test infrastructure).  `make -j` from the repo root.
NVCC ?= /usr/local/cuda/bin/nvcc
PKG := paper_2109_00626_b200
CSRC := $(PKG)/csrc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr -Xptxas -v
CU_SRCS := $(wildcard $(CSRC)/*.cu)
CPP_SRCS := $(wildcard $(CSRC)/*.cpp)
OBJS := $(patsubst $(CSRC)/%.cu,build/%.o,$(CU_SRCS)) $(patsubst $(CSRC)/%.cpp,build/%.o,$(CPP_SRCS))
HDRS := $(wildcard $(CSRC)/*.h) $(wildcard $(CSRC)/*.cuh) include/ttc.h

all: $(PKG)/libttc.so oracle/liboracle.so

build/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; exit 1)

build/%.o: $(CSRC)/%.cpp $(HDRS)
	@mkdir -p build
	$(NVCC) -O3 -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall -Xcompiler -O3 -x cu $(ARCH) -c $< -o $@

$(PKG)/libttc.so: $(OBJS)
	$(NVCC) -shared $(ARCH) -o $@ $(OBJS) -cudart static

oracle/liboracle.so: oracle/ttc_oracle.c
	gcc -O2 -fopenmp -fPIC -shared -o $@ $< -lm

clean:
	rm -rf build $(PKG)/libttc.so oracle/liboracle.so

.PHONY: all clean
