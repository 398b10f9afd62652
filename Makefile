# Builds the B200 product library paper_1601_07944_b200/libdg2d_b200.so
# (host setup C++ + sm_100a kernels + C ABI) and the test-only oracle.
NVCC ?= nvcc
CXX  := /usr/bin/g++
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -warn-spills
CXXFLAGS := -O2 -std=c++17 -fPIC -Wall -march=x86-64-v3
SRC := paper_1601_07944_b200/csrc
OBJ := build/obj
LIB := paper_1601_07944_b200/libdg2d_b200.so

DEV_OBJS  := $(OBJ)/kernels_p1.o $(OBJ)/kernels_p2.o $(OBJ)/kernels_p3.o $(OBJ)/kernels_p4.o $(OBJ)/kernels_p5.o $(OBJ)/solver.o
HOST_OBJS := $(OBJ)/basis.o $(OBJ)/mesh.o $(OBJ)/problems.o $(OBJ)/capi_setup.o
DEV_HDRS  := $(wildcard $(SRC)/device/*.cuh $(SRC)/device/*.hpp) include/dg2d_b200/dg2d_b200.h
HOST_HDRS := $(wildcard $(SRC)/host/*.hpp) include/dg2d_b200/dg2d_b200.h

all: $(LIB) oracle

$(LIB): $(DEV_OBJS) $(HOST_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^

$(OBJ)/%.o: $(SRC)/device/%.cu $(DEV_HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJ)/%.o: $(SRC)/host/%.cpp $(HOST_HDRS)
	@mkdir -p $(OBJ)
	$(CXX) $(CXXFLAGS) -c $< -o $@

oracle: $(LIB)
	$(MAKE) -C oracle liboracle.so
	@if [ -d /root/reference/proj ]; then $(MAKE) -C oracle ref && $(MAKE) -C oracle cpptest; fi

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
