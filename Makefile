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
CU_SRCS  := $(SRC)/store.cu $(SRC)/distance.cu $(SRC)/intersects.cu $(SRC)/pairs.cu $(SRC)/volume.cu $(SRC)/queries.cu $(SRC)/wkt.cu $(SRC)/host_copy.cu $(SRC)/group.cu $(SRC)/direct.cu $(SRC)/atiles.cu $(SRC)/capi.cu
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
	$(NVCC) $(ARCH) -shared -o $@ $^ -Xcompiler -fPIC -Xcompiler -pthread -lnccl

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

# The reference's own unit tests for the two replaced entry points
# (tests/test_{batch,volume,distance,intersect,geometry,store,sqlfe}.cpp, unmodified, compiled where
# they lie) with run_batch / mesh_volume routed to the device shim
# (tests/cpp/ref_route.hpp; test_sqlfe through the reference engine.cpp with
# engine.cpp:203 routed, tests/cpp/engine_route.hpp) and a minimal doctest
# stand-in. Test-only.
REFTESTS := test_batch test_volume test_distance test_intersect test_geometry test_store test_sqlfe
refunittest: $(LIB) oracle
	@if [ -d "$(REF)/include" ]; then \
	  mkdir -p $(BUILD)/refunit && \
	  for f in $(REFTESTS); do \
	    $(CXX) -std=c++20 -O2 -ffp-contract=off -Dtindb=tindb_ref -Itests/cpp/doctest_shim -I$(REF)/include -I$(REF)/tests \
	      -Iinclude -include tests/cpp/ref_route.hpp -c $(REF)/tests/$$f.cpp -o $(BUILD)/refunit/$$f.o || exit 1; done && \
	  $(CXX) -std=c++20 -O2 -ffp-contract=off -Dtindb=tindb_ref -I$(REF)/include -I$(REF)/tests \
	    -c $(REF)/tests/support/oracles.cpp -o $(BUILD)/refunit/oracles.o && \
	  $(CXX) -std=c++20 -O2 -DNDEBUG -ffp-contract=off -Dtindb=tindb_ref -I$(REF)/include -Iinclude \
	    -include tests/cpp/engine_route.hpp -c $(REF)/src/engine.cpp -o $(BUILD)/refunit/engine_routed.o && \
	  $(CXX) -std=c++20 -O2 -Itests/cpp/doctest_shim -c tests/cpp/ref_unit_main.cpp -o $(BUILD)/refunit/main.o && \
	  $(CXX) $(BUILD)/refunit/*.o -o $(BUILD)/ref_unit_tests -Loracle/_ref -ltindb_ref -L$(PKG) -ltindb_b200 \
	    -Wl,-rpath,'$$ORIGIN/../oracle/_ref' -Wl,-rpath,'$$ORIGIN/../$(PKG)'; \
	else echo "refunittest: $(REF) absent; keeping prebuilt $(BUILD)/ref_unit_tests"; fi

# The SQL route: the reference engine (engine.cpp, unmodified, force-including
# tests/cpp/engine_route.hpp) over the device shim, against the unmodified
# reference engine in oracle/_ref. Test-only binary; needs /root/reference.
ENGINE_SRCS := kernels batch wkt store sql_parser closure
enginetest: $(LIB) oracle
	@if [ -d "$(REF)/include" ]; then \
	  mkdir -p $(BUILD)/engine && \
	  for f in $(ENGINE_SRCS); do \
	    $(CXX) -std=c++20 -O2 -DNDEBUG -ffp-contract=off -fPIC -I$(REF)/include -c $(REF)/src/$$f.cpp \
	      -o $(BUILD)/engine/$$f.o || exit 1; done && \
	  $(CXX) -std=c++20 -O2 -DNDEBUG -ffp-contract=off -I$(REF)/include -Iinclude \
	    -include tests/cpp/engine_route.hpp -c $(REF)/src/engine.cpp -o $(BUILD)/engine/engine_routed.o && \
	  $(CXX) -std=c++20 -O2 -ffp-contract=off -I$(REF)/include -Iinclude -Itests/cpp \
	    -DENGINE_SIDE=engine_dev -DENGINE_SIDE_DEVICE -c tests/cpp/engine_side.cpp -o $(BUILD)/engine/side_dev.o && \
	  $(CXX) -std=c++20 -O2 -DNDEBUG -ffp-contract=off -Dtindb=tindb_ref -I$(REF)/include \
	    -include tests/cpp/engine_route_a17.hpp -c $(REF)/src/engine.cpp -o $(BUILD)/engine/engine_a17.o && \
	  $(CXX) -std=c++20 -O2 -ffp-contract=off -Dtindb=tindb_ref -I$(REF)/include -Itests/cpp \
	    -DENGINE_SIDE=engine_ref -c tests/cpp/engine_side.cpp -o $(BUILD)/engine/side_ref.o && \
	  $(CXX) -std=c++20 -O2 -Itests/cpp tests/cpp/engine_test.cpp $(BUILD)/engine/*.o -o $(BUILD)/engine_test \
	    -Loracle/_ref -ltindb_ref -L$(PKG) -ltindb_b200 -pthread \
	    -Wl,-rpath,'$$ORIGIN/../oracle/_ref' -Wl,-rpath,'$$ORIGIN/../$(PKG)'; \
	else echo "enginetest: $(REF) absent; keeping prebuilt $(BUILD)/engine_test"; fi

sass: $(LIB)
	cuobjdump -sass $(LIB) > $(BUILD)/libtindb_b200.sass

clean:
	rm -rf $(BUILD) $(LIB)
	$(MAKE) -C oracle clean

.PHONY: enginetest all lib oracle sass clean shimtest
