# Builds the sm_100a C-ABI library in-tree (it travels to the GPU box with
# the gpurun snapshot; git ignores *.so/*.o).
NVCC      ?= nvcc
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude \
             -Ipaper_1707_03268_b200/csrc --expt-relaxed-constexpr
SRC_DIR   := paper_1707_03268_b200/csrc
OBJ_DIR   := build/obj
LIB       := paper_1707_03268_b200/lib/libdpm_b200.so
SRCS      := $(wildcard $(SRC_DIR)/*.cu)
OBJS      := $(patsubst $(SRC_DIR)/%.cu,$(OBJ_DIR)/%.o,$(SRCS))
HDRS      := include/dpm_b200.h $(wildcard $(SRC_DIR)/*.cuh)

all: $(LIB)

$(OBJ_DIR)/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(OBJ_DIR)
	$(NVCC) $(NVFLAGS) $(EXTRA) -c $< -o $@

$(LIB): $(OBJS)
	@mkdir -p $(dir $(LIB))
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

# Checked build: device-side bounds checks (DPM_CHECK) compiled in; load it
# with DPM_LIB=paper_1707_03268_b200/lib/libdpm_b200_checked.so
CHK_DIR   := build/objc
CHK_LIB   := paper_1707_03268_b200/lib/libdpm_b200_checked.so
CHK_OBJS  := $(patsubst $(SRC_DIR)/%.cu,$(CHK_DIR)/%.o,$(SRCS))

$(CHK_DIR)/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(CHK_DIR)
	$(NVCC) $(NVFLAGS) -DDPM_CHECKED -c $< -o $@

$(CHK_LIB): $(CHK_OBJS)
	@mkdir -p $(dir $(CHK_LIB))
	$(NVCC) $(ARCH) -shared -o $@ $(CHK_OBJS)

checked: $(CHK_LIB)

ptxas: EXTRA := -Xptxas -v
ptxas: clean all

clean:
	rm -rf $(OBJ_DIR) $(LIB) $(CHK_DIR) $(CHK_LIB)

.PHONY: all clean ptxas checked
