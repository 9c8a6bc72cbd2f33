# Build recipe for the B200 GPUOS runtime.  Everything is compiled for sm_100a
# with nvcc (device code) or g++ (host code over the C-ABI).  `make` builds:
#   paper_2604_17861_b200/lib/libgpuos_cuda.so   device runtime + C-ABI
#   paper_2604_17861_b200/lib/libgpuos_bench.so  bench driver (bench.py)
#   build/cpp/test_runtime                       C++ runtime parity suite
#   oracle/liboracle.so                          CPU restatement (tests only)
#   oracle/_ref/*                                 reference built from /root/reference (when present)
NVCC ?= nvcc
CXX ?= g++
CC ?= gcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVEXTRA ?=
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude $(NVEXTRA)
CUDA_HOME ?= /usr/local/cuda
CXXFLAGS := -std=c++20 -O3 -ffp-contract=off -fPIC -Wall -Wno-unused-function -Iinclude -Ipaper_2604_17861_b200/include -isystem $(CUDA_HOME)/include
LIBDIR := paper_2604_17861_b200/lib
CSRC := paper_2604_17861_b200/csrc
OBJ := build/obj
DEV_HDRS := $(wildcard $(CSRC)/*.cuh) $(CSRC)/dev_state.h include/gpuos_ring_format.h include/gpuos_cuda.h
HOST_HDRS := $(wildcard paper_2604_17861_b200/include/gpuos/*.hpp) include/gpuos_cuda.h

all: lib bench cpp-tests oracle

lib: $(LIBDIR)/libgpuos_cuda.so $(LIBDIR)/gpuos_worker_rdc.cubin

# relocatable image of the same worker: native injected operators are linked
# against it at runtime (nvJitLink) into a new worker module
$(LIBDIR)/gpuos_worker_rdc.cubin: $(CSRC)/worker.cu $(DEV_HDRS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -O3 -std=c++17 -Iinclude -rdc=true -maxrregcount=80 -DGPUOS_WORKER_IMAGE -cubin $< -o $@
bench: $(LIBDIR)/libgpuos_bench.so
cpp-tests: build/cpp/test_runtime build/cpp/test_host build/cpp/gates

$(OBJ)/worker.o: $(CSRC)/worker.cu $(DEV_HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJ)/capi.o: $(CSRC)/capi.cu $(DEV_HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIBDIR)/libgpuos_cuda.so: $(OBJ)/worker.o $(OBJ)/capi.o
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -o $@ $^ -ldl

$(LIBDIR)/libgpuos_bench.so: tools/bench/gpuos_bench.cpp tools/bench/gpuos_bench_configs.cpp $(HOST_HDRS) $(LIBDIR)/libgpuos_cuda.so
	$(CXX) $(CXXFLAGS) -shared -o $@ tools/bench/gpuos_bench.cpp tools/bench/gpuos_bench_configs.cpp -L$(LIBDIR) -lgpuos_cuda -Wl,-rpath,'$$ORIGIN'

build/cpp/test_runtime: tests/cpp/test_runtime.cpp tests/cpp/check.hpp $(HOST_HDRS) $(LIBDIR)/libgpuos_cuda.so
	@mkdir -p build/cpp
	$(CXX) $(CXXFLAGS) -o $@ $< -L$(LIBDIR) -lgpuos_cuda -Wl,-rpath,'$$ORIGIN/../../$(LIBDIR)' -lpthread

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIBDIR)/*.so
	$(MAKE) -C oracle clean

.PHONY: all lib bench cpp-tests oracle clean

# acceptance gates C6/C8/C9/C10 + the reference bench workloads on the GPU runtime
build/cpp/gates: tools/bench/gpuos_gates.cpp $(HOST_HDRS) $(LIBDIR)/libgpuos_cuda.so
	@mkdir -p build/cpp
	$(CXX) $(CXXFLAGS) -o $@ $< -L$(LIBDIR) -lgpuos_cuda -Wl,-rpath,'$$ORIGIN/../../$(LIBDIR)' -lpthread

build/cpp/test_host: tests/cpp/test_host.cpp tests/cpp/check.hpp $(HOST_HDRS) $(LIBDIR)/libgpuos_cuda.so
	@mkdir -p build/cpp
	$(CXX) $(CXXFLAGS) -o $@ $< -L$(LIBDIR) -lgpuos_cuda -Wl,-rpath,'$$ORIGIN/../../$(LIBDIR)' -lpthread

# GPU-box probes (producer cost breakdown, finite worker generation for ncu,
# task-body call cost, PCIe round-trip floor)
probes: build/probe/submit_cost build/probe/profile_worker build/probe/body_bench build/probe/pingpong build/probe/burst_probe
build/probe/body_bench: tools/probe/body_bench.cu $(DEV_HDRS)
	@mkdir -p build/probe
	$(NVCC) $(ARCH) -O3 -std=c++17 -Iinclude -I$(CSRC) -o $@ $<
build/probe/pingpong: tools/probe/pingpong.cu
	@mkdir -p build/probe
	$(NVCC) $(ARCH) -O3 -o $@ $<
build/probe/%: tools/probe/%.cpp $(HOST_HDRS) $(LIBDIR)/libgpuos_cuda.so
	@mkdir -p build/probe
	$(CXX) $(CXXFLAGS) -o $@ $< -L$(LIBDIR) -lgpuos_cuda -Wl,-rpath,'$$ORIGIN/../../$(LIBDIR)' -lpthread
# latency-bisection build of the runtime (clock64 stamps between pipeline
# points, printed by the completer): build/dbg/libgpuos_cuda.so, used by
# tools/lat_stamps.sh in place of the product library on the GPU box
lat-debug:
	$(MAKE) lib NVEXTRA=-DGPUOS_LAT_STAMPS OBJ=build/dbg LIBDIR=build/dbg
# fetcher hand-off cycle profile (build/fprof/libgpuos_cuda.so, swapped in by tools/fetch_prof.sh)
fetch-prof:
	$(MAKE) lib NVEXTRA=-DGPUOS_FETCH_PROF OBJ=build/fprof LIBDIR=build/fprof
.PHONY: probes lat-debug fetch-prof
