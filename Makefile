# Top-level build: the B200 C-ABI library and the C++ host library.
#   make            -> paper_2311_18141_b200/lib/librdmm_cuda.so (+ oracle)
# All device code is compiled for sm_100a only.
NVCC    ?= /usr/local/cuda/bin/nvcc
PKG     := paper_2311_18141_b200
SRC     := $(PKG)/csrc
OBJ     := build/obj
LIBDIR  := $(PKG)/lib
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 \
           -Iinclude -I$(SRC) --expt-relaxed-constexpr -Xptxas -warn-spills
CUDA_SRCS := $(wildcard $(SRC)/*.cu)
CUDA_OBJS := $(patsubst $(SRC)/%.cu,$(OBJ)/%.o,$(CUDA_SRCS))
CXX_SRCS  := $(wildcard $(SRC)/*.cpp)
CXX_OBJS  := $(patsubst $(SRC)/%.cpp,$(OBJ)/%.cpp.o,$(CXX_SRCS))
CXX       := g++
CXXFLAGS  := -std=c++20 -O2 -g -fPIC -Wall -Wno-unused-function -Iinclude -I$(SRC) -pthread
HDRS := $(wildcard include/*.h) $(wildcard include/rdmm/*.hpp) $(wildcard $(SRC)/*.cuh) $(wildcard $(SRC)/*.h)

all: $(LIBDIR)/librdmm_cuda.so oracle build/tests/test_api

$(OBJ)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJ)/%.cpp.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJ)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIBDIR)/librdmm_cuda.so: $(CUDA_OBJS) $(CXX_OBJS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(CUDA_OBJS) $(CXX_OBJS) -lpthread -lrt -ldl -lz

# C++ drop-in API test program (run on the GPU by tests/test_cpp_gpu.py)
build/tests/test_api: tests/cpp/test_api.cpp $(LIBDIR)/librdmm_cuda.so $(HDRS)
	@mkdir -p build/tests
	$(CXX) -std=c++20 -O1 -g -Iinclude -pthread -o $@ tests/cpp/test_api.cpp \
	    -L$(LIBDIR) -lrdmm_cuda -Wl,-rpath,'$$ORIGIN/../../$(LIBDIR)'

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf build $(LIBDIR)

.PHONY: all oracle clean
