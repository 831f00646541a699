# Build for B200 (sm_100a) only.
#   make            -> paper_2512_21967_b200/libblest_b200.so (product) + oracle libs (checkers)
#   make lib        -> product library only
NVCC      ?= /usr/local/cuda/bin/nvcc
CUDA_HOME ?= /usr/local/cuda
ARCH      := -gencode arch=compute_100a,code=sm_100a
NVFLAGS   := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr
SRC_DIR   := paper_2512_21967_b200/csrc
OBJ_DIR   := build/obj
SRCS      := $(wildcard $(SRC_DIR)/*.cu)
OBJS      := $(patsubst $(SRC_DIR)/%.cu,$(OBJ_DIR)/%.o,$(SRCS))
HDRS      := $(wildcard $(SRC_DIR)/*.cuh) include/blest_b200.h
LIB       := paper_2512_21967_b200/libblest_b200.so

all: lib oracle

lib: $(LIB)

$(OBJ_DIR)/%.o: $(SRC_DIR)/%.cu $(HDRS)
	@mkdir -p $(OBJ_DIR)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(OBJ_DIR)/$*.ptxas.txt || (cat $(OBJ_DIR)/$*.ptxas.txt; false)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart

oracle:
	$(MAKE) -s -C oracle all

clean:
	rm -rf build $(LIB)

.PHONY: all lib oracle clean cpptest

cpptest: tests/cpp/facade_test

# the facade test program takes its expected values from the compiled reference (oracle/_ref)
tests/cpp/facade_test: tests/cpp/facade_test.cpp include/blest_b200.hpp include/blest_b200.h $(LIB) | oracle/_ref/libblest_ref.so
	g++ -std=c++20 -O2 -Wall -Iinclude -I$(CUDA_HOME)/include -o $@ tests/cpp/facade_test.cpp -Lpaper_2512_21967_b200 -lblest_b200 \
	    -Loracle/_ref -lblest_ref -L$(CUDA_HOME)/lib64 -lcudart -pthread \
	    -Wl,-rpath,'$$ORIGIN/../../paper_2512_21967_b200' -Wl,-rpath,'$$ORIGIN/../../oracle/_ref'

oracle/_ref/libblest_ref.so:
	$(MAKE) -s -C oracle ref
