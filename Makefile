# Builds the product library (sm_100a) and the CPU oracle.
#   make            -> paper_1304_4453_b200/libcommdet_cuda.so + oracle
#   make lib        -> product only
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH ?= -gencode arch=compute_100a,code=sm_100a
NVFLAGS = -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
          --expt-relaxed-constexpr -Iinclude -Xptxas -warn-spills
SRC_DIR = paper_1304_4453_b200/csrc
OBJ_DIR = build/obj
SRCS = $(wildcard $(SRC_DIR)/*.cu)
OBJS = $(patsubst $(SRC_DIR)/%.cu,$(OBJ_DIR)/%.o,$(SRCS))
HDRS = $(wildcard $(SRC_DIR)/*.cuh) include/commdet_cuda.h
LIB = paper_1304_4453_b200/libcommdet_cuda.so

all: lib shim cli oracle

lib: $(LIB)

# reference-style C++ caller of the drop-in shim (include/commdet/gpu.hpp)
SHIM = build/shim_kat
shim: $(SHIM)
$(SHIM): tests/cpp/shim_kat.cpp include/commdet/gpu.hpp include/commdet_cuda.h $(LIB)
	@mkdir -p build
	g++ -std=c++20 -O2 -Iinclude tests/cpp/shim_kat.cpp -o $@ -Lpaper_1304_4453_b200 -lcommdet_cuda \
	    -Wl,-rpath,'$$ORIGIN/../paper_1304_4453_b200'

# the reference CLI's drop-in (tools/commdet_gpu.cpp over the shim)
CLI = build/commdet_gpu
cli: $(CLI)
$(CLI): tools/commdet_gpu.cpp include/commdet/gpu.hpp include/commdet_cuda.h $(LIB)
	@mkdir -p build
	g++ -std=c++20 -O2 -Iinclude tools/commdet_gpu.cpp -o $@ -Lpaper_1304_4453_b200 -lcommdet_cuda \
	    -Wl,-rpath,'$$ORIGIN/../paper_1304_4453_b200'

$(OBJ_DIR)/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(OBJ_DIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -Xcompiler -fPIC

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all lib shim oracle clean
