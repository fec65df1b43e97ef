# Builds the C-ABI shared library of the B200 engine (sm_100a only).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
CSRC := paper_2204_10319_b200/csrc
SRCS := $(CSRC)/capi.cu $(CSRC)/mapping.cu $(CSRC)/movement.cu $(CSRC)/gemm_sm100.cu \
        $(CSRC)/implicit_sm100.cu $(CSRC)/voxelize.cu $(CSRC)/reorder.cu \
        $(CSRC)/upconv_sm100.cu
OBJS := $(patsubst $(CSRC)/%.cu,build/%.o,$(SRCS))
LIB  := paper_2204_10319_b200/libsparseconv_b200.so
FLAGS := -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC -Iinclude -Xptxas -v

all: $(LIB)

build/%.o: $(CSRC)/%.cu $(CSRC)/common.cuh $(CSRC)/sm100_ptx.cuh include/sparseconv_b200.h
	@mkdir -p build
	$(NVCC) $(FLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

# per-stage timeline build of the fused conv (tools/ic_trace.py); not shipped
TRACE_LIB := paper_2204_10319_b200/libsparseconv_b200_trace.so
trace: $(TRACE_LIB)
$(TRACE_LIB): $(SRCS) $(CSRC)/common.cuh $(CSRC)/sm100_ptx.cuh include/sparseconv_b200.h
	@mkdir -p build/trace
	for f in $(SRCS); do b=$$(basename $$f .cu); \
	  $(NVCC) $(FLAGS) -DSCB_IC_TRACE -c $$f -o build/trace/$$b.o 2> build/trace/$$b.log || exit 1; done
	$(NVCC) $(ARCH) -shared -o $@ build/trace/*.o

clean:
	rm -rf build $(LIB)

.PHONY: all clean trace
