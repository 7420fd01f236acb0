# tindb_b200: sm_100a engine (C ABI shared library) + test-only oracle.
#
#   make            -> paper_1808_09571_b200/libtindb_b200.so, oracle libs
#   make lib        -> only the product library
#   make sass       -> cuobjdump -sass of the kernels into build/
NVCC     ?= /usr/local/cuda/bin/nvcc
CXX      ?= g++
ARCH     := -gencode arch=compute_100a,code=sm_100a
PKG      := paper_1808_09571_b200
SRC      := $(PKG)/csrc
BUILD    := build
LIB      := $(PKG)/libtindb_b200.so
CU_SRCS  := $(SRC)/store.cu $(SRC)/distance.cu $(SRC)/intersects.cu $(SRC)/pairs.cu $(SRC)/volume.cu $(SRC)/queries.cu $(SRC)/wkt.cu $(SRC)/host_copy.cu $(SRC)/capi.cu
CU_OBJS  := $(patsubst $(SRC)/%.cu,$(BUILD)/%.o,$(CU_SRCS))
CPP_OBJS := $(BUILD)/generators.o
HDRS     := $(wildcard $(SRC)/*.h $(SRC)/*.cuh) include/tindb_b200.h
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v -Iinclude -I$(SRC) \
            --expt-relaxed-constexpr $(EXTRA)
CXXFLAGS := -O2 -fPIC -std=c++17 -ffp-contract=off -Iinclude

all: lib oracle

lib: $(LIB)

$(BUILD):
	mkdir -p $(BUILD)

$(BUILD)/%.o: $(SRC)/%.cu $(HDRS) | $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(BUILD)/$*.ptxas.txt || (cat $(BUILD)/$*.ptxas.txt; false)

$(BUILD)/generators.o: $(SRC)/generators.cpp include/tindb_b200.h | $(BUILD)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB): $(CU_OBJS) $(CPP_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -Xcompiler -fPIC -Xcompiler -pthread

oracle:
	$(MAKE) -C oracle

# C++ shim (include/tindb_b200/kernels.hpp) against the reference's own types
# and dispatch; only buildable where /root/reference exists (the binary then
# travels to the GPU box with the snapshot).
REF ?= /root/reference/proj
shimtest: $(LIB) oracle
	@if [ -d "$(REF)/include" ]; then \
	  $(CXX) -std=c++20 -O2 -ffp-contract=off -Dtindb=tindb_ref -I$(REF)/include -Iinclude \
	    tests/cpp/shim_test.cpp -o $(BUILD)/shim_test -Loracle/_ref -ltindb_ref -L$(PKG) -ltindb_b200 \
	    -Wl,-rpath,'$$ORIGIN/../oracle/_ref' -Wl,-rpath,'$$ORIGIN/../$(PKG)'; \
	else echo "shimtest: $(REF) absent; keeping prebuilt $(BUILD)/shim_test"; fi

sass: $(LIB)
	cuobjdump -sass $(LIB) > $(BUILD)/libtindb_b200.sass

clean:
	rm -rf $(BUILD) $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all lib oracle sass clean shimtest
