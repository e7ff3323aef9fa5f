# Builds libsccl_exec.so (C++ host + sm_100a kernels) in-tree and the CPU oracle.
CUDA ?= /usr/local/cuda
NVCC ?= $(CUDA)/bin/nvcc
CXX ?= g++
PKG := paper_2008_08708_b200
SRC := $(PKG)/csrc
OBJ := build/obj
LIB := $(PKG)/lib/libsccl_exec.so
CLI := $(PKG)/lib/sccl-exec
ARCH := -gencode arch=compute_100a,code=sm_100a
CXXFLAGS := -O2 -std=c++17 -fPIC -Wall -Wextra -Wno-unused-parameter -ffp-contract=off -I$(CUDA)/include -Iinclude
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xptxas -v -Iinclude

HOST_SRCS := $(wildcard $(SRC)/sccl/*.cpp)
CU_SRCS := $(wildcard $(SRC)/kernels/*.cu)
HDRS := $(wildcard $(SRC)/sccl/*.hpp) $(wildcard include/*.h)
HOST_OBJS := $(patsubst $(SRC)/sccl/%.cpp,$(OBJ)/%.o,$(HOST_SRCS))
CU_OBJS := $(patsubst $(SRC)/kernels/%.cu,$(OBJ)/%.cu.o,$(CU_SRCS))

all: $(LIB) $(CLI) oracle

$(OBJ)/%.o: $(SRC)/sccl/%.cpp $(HDRS)
	@mkdir -p $(OBJ)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OBJ)/%.cu.o: $(SRC)/kernels/%.cu $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJ)/$*.ptxas.txt || (cat $(OBJ)/$*.ptxas.txt; false)

$(LIB): $(HOST_OBJS) $(CU_OBJS)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $^ -lpthread

$(CLI): $(SRC)/tools/sccl_exec_cli.cpp $(LIB) include/sccl_exec.h
	$(CXX) -O2 -std=c++17 -I$(CUDA)/include -Iinclude $< -o $@ -L$(PKG)/lib -lsccl_exec -L$(CUDA)/lib64 -lcudart -Wl,-rpath,'$$ORIGIN' -Wl,-rpath,$(CUDA)/lib64

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf build $(LIB) $(CLI)
	$(MAKE) -s -C oracle clean

.PHONY: all oracle clean
