# Builds the product library (host C++ engine + sm_100a kernels behind the C ABI)
# and the CPU oracle. `python -c "import __graft_entry__ as g; g.build()"` runs this.
NVCC      ?= /usr/local/cuda/bin/nvcc
CXX       ?= g++
PKG       := paper_2602_21597_b200
BUILD     := build
LIBDIR    := $(PKG)/_lib
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Xptxas -v
CXXFLAGS  := -O3 -std=c++20 -fPIC -Wall -Wextra -Iinclude

HOST_SRC  := $(wildcard $(PKG)/csrc/host/*.cpp)
CUDA_SRC  := $(wildcard $(PKG)/csrc/cuda/*.cu)
HOST_OBJ  := $(patsubst $(PKG)/csrc/host/%.cpp,$(BUILD)/host/%.o,$(HOST_SRC))
CUDA_OBJ  := $(patsubst $(PKG)/csrc/cuda/%.cu,$(BUILD)/cuda/%.o,$(CUDA_SRC))
HEADERS   := $(wildcard include/ngdb/*.hpp include/ngdb/*.h) $(wildcard $(PKG)/csrc/cuda/*.cuh)

LIB       := $(LIBDIR)/libngdb_b200.so

.PHONY: all lib oracle examples clean
all: lib oracle examples

# C++ driver of the row-sharded step (no Python): links the product library
EXAMPLES := $(LIBDIR)/sharded_train
examples: $(EXAMPLES)
$(LIBDIR)/sharded_train: tools/cpp/sharded_train.cpp $(LIB) $(HEADERS)
	$(CXX) $(CXXFLAGS) $< -o $@ -L$(LIBDIR) -lngdb_b200 -Wl,-rpath,'$$ORIGIN'

lib: $(LIB)

$(BUILD)/host/%.o: $(PKG)/csrc/host/%.cpp $(HEADERS)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(BUILD)/cuda/%.o: $(PKG)/csrc/cuda/%.cu $(HEADERS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/cuda/$*.ptxas.log || (cat $(BUILD)/cuda/$*.ptxas.log; exit 1)

$(LIB): $(HOST_OBJ) $(CUDA_OBJ)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -o $@ $(HOST_OBJ) $(CUDA_OBJ) -lpthread

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf $(BUILD) $(LIBDIR)/*.so
	$(MAKE) -C oracle clean
