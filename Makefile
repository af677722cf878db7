# Builds the B200 engine as an in-tree shared library (sm_100a) and the
# oracle's C pieces (none yet).  `python -c "import __graft_entry__ as g; g.build()"`
# runs the same recipe.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -lineinfo -std=c++17 $(ARCH) -Xcompiler -fPIC -Xcompiler -g -Xptxas -v --expt-relaxed-constexpr
SRC := $(wildcard paper_2506_04732_b200/csrc/*.cu)
HDR := $(wildcard paper_2506_04732_b200/csrc/*.h) $(wildcard paper_2506_04732_b200/csrc/*.cuh) include/t2s2.h
LIB := paper_2506_04732_b200/lib/libt2s2.so
OBJ := $(patsubst paper_2506_04732_b200/csrc/%.cu,build/%.o,$(SRC))

all: $(LIB)

build/%.o: paper_2506_04732_b200/csrc/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJ)
	@mkdir -p paper_2506_04732_b200/lib
	$(NVCC) $(ARCH) -shared -Xcompiler -fPIC -o $@ $(OBJ) -lcudart

clean:
	rm -rf build $(LIB)

.PHONY: all clean
