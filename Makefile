# Builds the sm_100a FP64 PowerURV library (C ABI: include/urv_b200.h).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Iinclude --expt-relaxed-constexpr
SRC_DIR := paper_1812_06007_b200/csrc
SRCS := $(SRC_DIR)/dgemm.cu $(SRC_DIR)/qr.cu $(SRC_DIR)/rng.cu $(SRC_DIR)/svd.cu $(SRC_DIR)/io.cu $(SRC_DIR)/profile.cu $(SRC_DIR)/xfer.cu $(SRC_DIR)/comm.cu $(SRC_DIR)/urv.cu
HDRS := $(wildcard $(SRC_DIR)/*.h $(SRC_DIR)/*.cuh) include/urv_b200.h
OBJS := $(patsubst $(SRC_DIR)/%.cu,build/%.o,$(SRCS))
LIB := paper_1812_06007_b200/liburv_b200.so

all: $(LIB)

build/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJS) -ldl

clean:
	rm -rf build $(LIB)

.PHONY: all clean
