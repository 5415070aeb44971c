# Builds the B200 (sm_100a) C-ABI library in-tree so it travels with gpurun.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3
SRC := $(wildcard paper_1908_02721_b200/csrc/*.cu)
HDR := $(wildcard paper_1908_02721_b200/csrc/*.cuh) include/fasttt_b200.h
OBJ := $(patsubst paper_1908_02721_b200/csrc/%.cu,build/%.o,$(SRC))
LIB := paper_1908_02721_b200/libfasttt_b200.so

all: $(LIB)

build/%.o: paper_1908_02721_b200/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJ)

ptxas:
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $(SRC) -o /dev/null

clean:
	rm -rf build $(LIB)

.PHONY: all clean ptxas
