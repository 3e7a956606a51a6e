# wavepipe-b200 build: one in-tree shared library with the C ABI.
#   paper_2308_15762_b200/libwavepipe.so
# Host code: g++ C++20.  Device code: nvcc for sm_100a only.
CUDA     ?= /usr/local/cuda
NVCC     ?= $(CUDA)/bin/nvcc
CXX      ?= g++
PKG      := paper_2308_15762_b200
CSRC     := $(PKG)/csrc
OBJ      := build/obj
LIB      := $(PKG)/libwavepipe.so

INCLUDES := -Iinclude -I$(CSRC) -I$(CUDA)/include
CXXFLAGS := -std=c++20 -O2 -fPIC -ffp-contract=off -Wall -Wextra $(INCLUDES)
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(EXTRA_NVFLAGS) -std=c++20 -O3 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -ffp-contract=off \
            --expt-relaxed-constexpr -Xptxas -v $(INCLUDES)

CORE_SRCS := $(wildcard $(CSRC)/core/*.cpp) $(wildcard $(CSRC)/*.cpp) $(wildcard $(CSRC)/runtime/*.cpp)
CU_SRCS   := $(wildcard $(CSRC)/kernels/*.cu)
CORE_OBJS := $(patsubst $(CSRC)/%.cpp,$(OBJ)/%.o,$(CORE_SRCS))
CU_OBJS   := $(patsubst $(CSRC)/%.cu,$(OBJ)/%.cu.o,$(CU_SRCS))
HDRS      := $(wildcard include/*.h include/wavepipe/*.hpp $(CSRC)/*.hpp $(CSRC)/*/*.hpp $(CSRC)/*/*.cuh)

all: $(LIB)

$(OBJ)/%.o: $(CSRC)/%.cpp $(HDRS)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OBJ)/%.cu.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; exit 1)

$(LIB): $(CORE_OBJS) $(CU_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -L$(CUDA)/lib64 -lcudart_static -ldl -lpthread -lrt

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)

.PHONY: all clean oracle
