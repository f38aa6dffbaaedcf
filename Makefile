# Build of the B200-native Oases TMP hot path.
#   make            -> paper_2305_16121_b200/liboases.so (C-ABI) + _core python module
#   make oracle     -> oracle/build/liboracle.so (fp64 restatement, test-only)
#   make ref        -> oracle/_ref/* (the reference built from /root/reference, test-only)
CUDA    ?= /usr/local/cuda
NVCC    ?= $(CUDA)/bin/nvcc
CXX     := /usr/bin/g++
PYTHON  ?= python
PKG     := paper_2305_16121_b200
SRC     := $(PKG)/csrc
BUILD   := build
JSON_INC ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
# NCCL: the build links the same libnccl.so.2 torch loads (the nvidia-nccl wheel,
# 2.28.x) and records its directory as rpath, so the process has ONE NCCL no
# matter whether torch or liboases is imported first (the system 2.27 lacks
# symbols libtorch_cuda needs).
NCCL_DIR ?= $(shell $(PYTHON) -c "import nvidia.nccl, os; print(list(nvidia.nccl.__path__)[0])" 2>/dev/null)
ifeq ($(NCCL_DIR),)
NCCL_INC := /usr/include
NCCL_LINK := -lnccl
else
NCCL_INC := $(NCCL_DIR)/include
NCCL_LINK := -L$(NCCL_DIR)/lib -l:libnccl.so.2 -Xlinker -rpath,$(NCCL_DIR)/lib
endif
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -ccbin /usr/bin/g++ -std=c++17 -O3 -lineinfo $(ARCH) -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr -Iinclude -I$(NCCL_INC)
CXXFLAGS := -std=c++20 -O2 -fPIC -Wall -Wextra -Iinclude -I$(NCCL_INC) -I$(CUDA)/include -I$(JSON_INC)

CU_SRCS  := $(wildcard $(SRC)/kernels/*.cu) $(wildcard $(SRC)/runtime/*.cu)
CPP_SRCS := $(wildcard $(SRC)/host/*.cpp) $(wildcard $(SRC)/runtime/*.cpp)
CU_OBJS  := $(patsubst $(SRC)/%.cu,$(BUILD)/%.o,$(CU_SRCS))
CPP_OBJS := $(patsubst $(SRC)/%.cpp,$(BUILD)/%.o,$(CPP_SRCS))
LIB      := $(PKG)/liboases.so
PYEXT    := $(shell $(PYTHON) -c "import sysconfig;print(sysconfig.get_config_var('EXT_SUFFIX'))")
CORE     := $(PKG)/_core$(PYEXT)
PYBIND_INC := $(shell $(PYTHON) -m pybind11 --includes)

all: $(LIB) $(CORE)

$(BUILD)/%.o: $(SRC)/%.cu $(wildcard $(SRC)/kernels/*.cuh $(SRC)/kernels/*.h $(SRC)/runtime/*.h include/*.h include/oases/*.hpp)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; false)

$(BUILD)/%.o: $(SRC)/%.cpp $(wildcard $(SRC)/runtime/*.h $(SRC)/host/*.h include/*.h include/oases/*.hpp)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB): $(CU_OBJS) $(CPP_OBJS)
	$(NVCC) -ccbin /usr/bin/g++ -shared $(ARCH) -o $@ $^ -L$(CUDA)/lib64 -lcudart -Xlinker -rpath,$(CUDA)/lib64 $(NCCL_LINK)

$(CORE): $(SRC)/python/bindings.cpp $(LIB) include/oases/tmpsim.hpp include/oases/runtime.hpp
	$(CXX) -std=c++20 -O2 -shared -fPIC $(PYBIND_INC) -Iinclude -I$(CUDA)/include -I$(JSON_INC) $< -o $@ \
	  -L$(PKG) -loases -Wl,-rpath,'$$ORIGIN'

oracle:
	$(MAKE) -C oracle

ref:
	$(MAKE) -C oracle ref

clean:
	rm -rf $(BUILD) $(LIB) $(PKG)/_core*.so

.PHONY: all oracle ref clean
