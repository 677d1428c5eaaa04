# Builds libgx.so (CUDA kernels for sm_100a + C++ runtime/planner behind the C ABI in
# include/gx.h) in-tree, plus the test-only oracle artefacts under oracle/.
#
#   make            -> paper_2211_13878_b200/libgx.so
#   make oracle     -> oracle/_ref/libparplan_ref.so (reference planner, test-only)
PKG      := paper_2211_13878_b200
CSRC     := $(PKG)/csrc
BUILD    := build
NVCC     ?= nvcc
CXX      ?= g++
VENV_SP  := $(shell python -c "import site,sys; print(site.getsitepackages()[0])" 2>/dev/null)
NCCL_DIR := $(VENV_SP)/nvidia/nccl
JSON_INC := $(VENV_SP)/include/cudnn_frontend/thirdparty
CUDA_HOME ?= /usr/local/cuda

ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
            -Iinclude -I$(CSRC)/kernels -I$(NCCL_DIR)/include --expt-relaxed-constexpr
# The plan/search code must reproduce the reference's floating-point results bit for bit:
# no fast-math, no FMA contraction, no -march=native (SURVEY.md §7 hard part 1).
CXXFLAGS := -std=c++20 -O2 -fPIC -ffp-contract=off -fvisibility=hidden -Wall -Wextra \
            -Iinclude -I$(CSRC)/kernels -I$(CSRC)/third_party -I$(JSON_INC) -I$(NCCL_DIR)/include -I$(CUDA_HOME)/include

CU_SRCS  := $(wildcard $(CSRC)/kernels/*.cu)
CC_SRCS  := $(wildcard $(CSRC)/runtime/*.cc) $(wildcard $(CSRC)/parplan/*.cc)
CU_OBJS  := $(patsubst $(CSRC)/%.cu,$(BUILD)/%.o,$(CU_SRCS))
CC_OBJS  := $(patsubst $(CSRC)/%.cc,$(BUILD)/%.o,$(CC_SRCS))
HDRS     := $(wildcard include/*.h include/parplan/*.h $(CSRC)/kernels/*.cuh $(CSRC)/kernels/*.h $(CSRC)/runtime/*.h)

LIB      := $(PKG)/libgx.so

CLI      := $(PKG)/parplan
CLI_OBJS := $(BUILD)/tools/parplan_cli.o $(filter-out %plan_capi.o,$(filter $(BUILD)/parplan/%,$(CC_OBJS)))

all: $(LIB) $(CLI)

$(BUILD)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(BUILD)/%.o: $(CSRC)/%.cc $(HDRS)
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB): $(CU_OBJS) $(CC_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -Xlinker -rpath=$(NCCL_DIR)/lib \
	    -L$(NCCL_DIR)/lib -l:libnccl.so.2 -lpthread

# The `parplan` command line (reference proj/tools/parplan_main.cc): links the planner objects
# statically and dlopens libgx.so (next to it) only for `run` / `profile`.
$(CLI): $(CLI_OBJS)
	$(CXX) -o $@ $^ -ldl -lpthread

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf $(BUILD) $(LIB) $(CLI)

.PHONY: all oracle clean
