# Builds the sm_100a solver library in-tree (it travels to the GPU box).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC -Xptxas -v
SRC := $(wildcard paper_1302_6945_b200/csrc/*.cu)
OBJ := $(patsubst paper_1302_6945_b200/csrc/%.cu,build/%.o,$(SRC))
LIB := paper_1302_6945_b200/libtoepreg_b200.so

all: $(LIB)

build/%.o: paper_1302_6945_b200/csrc/%.cu paper_1302_6945_b200/csrc/*.cuh include/toepreg_b200.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart

clean:
	rm -rf build $(LIB)

.PHONY: all clean
