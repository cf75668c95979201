# Build of the B200-native engine (sm_100a) and its test-only checkers.
#   make            -> paper_1801_00338_b200/libbfly_b200.so (+ libbfly_synth.so, oracle)
#   make lib        -> only the CUDA engine
NVCC ?= nvcc
PKG := paper_1801_00338_b200
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall \
           --expt-relaxed-constexpr -Xptxas -warn-spills
CU_SRCS := $(wildcard $(PKG)/csrc/*.cu)
CU_OBJS := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(CU_SRCS))
HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/bfly_b200.h

all: lib synth oracle

lib: $(PKG)/libbfly_b200.so

build/%.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(PKG)/libbfly_b200.so: $(CU_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(CU_OBJS) -lcudart

synth: $(PKG)/libbfly_synth.so

$(PKG)/libbfly_synth.so: $(PKG)/synth/synth.cpp $(PKG)/synth/synth.h
	g++ -O3 -march=x86-64-v2 -std=c++17 -fPIC -shared -Wall -o $@ $< -lpthread

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(PKG)/libbfly_b200.so $(PKG)/libbfly_synth.so
	$(MAKE) -C oracle clean

.PHONY: all lib synth oracle clean
