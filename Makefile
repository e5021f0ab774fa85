# Builds the three libraries of the repo (see __graft_entry__.build()).
#   paper_2410_17226_b200/libcbfs.so  — the product (CUDA, sm_100a)
#   oracle/liboracle.so               — CPU oracle (test infrastructure only)
#   cbfs_inputs/libcbfsgen.so         — seeded input generators (shared)
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -std=c++17 $(ARCH) -O3 -lineinfo -Xcompiler -fPIC -Xptxas -v
CSRC := paper_2410_17226_b200/csrc
SRCS := $(CSRC)/graph.cu $(CSRC)/cbfs.cu $(CSRC)/sparse.cu $(CSRC)/select.cu $(CSRC)/query.cu $(CSRC)/labels.cu $(CSRC)/pll.cu $(CSRC)/digest.cu
OBJS := $(patsubst $(CSRC)/%.cu,build/%.o,$(SRCS))

all: paper_2410_17226_b200/libcbfs.so oracle/liboracle.so cbfs_inputs/libcbfsgen.so

build/%.o: $(CSRC)/%.cu $(CSRC)/common.cuh $(CSRC)/engine.cuh include/cbfs.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

paper_2410_17226_b200/libcbfs.so: $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart

oracle/liboracle.so: oracle/oracle.c
	gcc -O2 -std=c11 -fPIC -shared -pthread $< -o $@

cbfs_inputs/libcbfsgen.so: cbfs_inputs/gen.c include/cbfs_gen.h
	gcc -O2 -std=c11 -fPIC -shared -pthread $< -o $@ -lm

clean:
	rm -rf build paper_2410_17226_b200/libcbfs.so oracle/liboracle.so cbfs_inputs/libcbfsgen.so

.PHONY: all clean
