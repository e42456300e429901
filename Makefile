# SPDX-License-Identifier: Apache-2.0
# Builds the B200 product library (sm_100a) and the CPU oracle.
#   make            -> paper_2504_17449_b200/_lib/libhmi_b200.so + oracle/_build/liboracle.so
#   make ref        -> oracle/_ref/libhmiref.so (needs /root/reference; see oracle/build_ref.sh)
#   make cppapi     -> cpp_api/_build/libhmi_cuda_backend.a (hmi::sched::CudaBackend, compiled
#                      against the reference's public headers) + its test program, linked with
#                      the reference library oracle/_ref builds (needs /root/reference)
NVCC     ?= /usr/local/cuda/bin/nvcc
CXX      ?= g++
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall \
            --expt-relaxed-constexpr -Xptxas -v
CSRC     := paper_2504_17449_b200/csrc
LIBDIR   := paper_2504_17449_b200/_lib
OBJDIR   := build/obj
CU_SRCS  := $(wildcard $(CSRC)/*.cu)
CPP_SRCS := $(wildcard $(CSRC)/*.cpp)
OBJS     := $(patsubst $(CSRC)/%.cu,$(OBJDIR)/%.o,$(CU_SRCS)) \
            $(patsubst $(CSRC)/%.cpp,$(OBJDIR)/%.cpp.o,$(CPP_SRCS))
HDRS     := $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.hpp) include/hmi_gpu.h

all: $(LIBDIR)/libhmi_b200.so oracle

$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJDIR)/$*.ptxas.log || (cat $(OBJDIR)/$*.ptxas.log; false)

$(OBJDIR)/%.cpp.o: $(CSRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) -O3 -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall -x cu $(ARCH) -c $< -o $@

$(LIBDIR)/libhmi_b200.so: $(OBJS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -cudart static -lpthread

oracle:
	$(MAKE) -C oracle

ref:
	bash oracle/build_ref.sh

REF_INC  ?= /root/reference/proj/include
CPP_OUT  := cpp_api/_build
CPPFLAGS_API := -std=c++20 -O2 -Wall -include mutex -I$(REF_INC) -Icpp_api -Iinclude

cppapi: $(CPP_OUT)/libhmi_cuda_backend.a $(CPP_OUT)/test_cuda_backend

$(CPP_OUT)/cuda_backend.o: cpp_api/cuda_backend.cpp cpp_api/hmi/scheduler/cuda_backend.hpp include/hmi_gpu.h
	@mkdir -p $(CPP_OUT)
	$(CXX) $(CPPFLAGS_API) -fPIC -c $< -o $@

$(CPP_OUT)/libhmi_cuda_backend.a: $(CPP_OUT)/cuda_backend.o
	ar rcs $@ $^

$(CPP_OUT)/test_cuda_backend: tests/cpp/test_cuda_backend.cpp $(CPP_OUT)/libhmi_cuda_backend.a \
		$(LIBDIR)/libhmi_b200.so oracle/_ref/libhmiref.so
	$(CXX) $(CPPFLAGS_API) $< -o $@ $(CPP_OUT)/libhmi_cuda_backend.a -Loracle/_ref -lhmiref \
		-L$(LIBDIR) -lhmi_b200 -Wl,-rpath,'$$ORIGIN/../../oracle/_ref' \
		-Wl,-rpath,'$$ORIGIN/../../$(LIBDIR)' -lpthread

clean:
	rm -rf build $(LIBDIR)

.PHONY: all oracle ref cppapi clean
