# Build recipe for the B200 PipeTransformer hot path.
#   make lib     -> paper_2102_03161_b200/libeps_b200.so  (product: control plane + sm_100a kernels)
#   make oracle  -> oracle/_ref/libeps_ref.so              (checker: the reference's own sources)
# __graft_entry__.build() runs both.  nvcc cross-compiles sm_100a without a GPU.

NVCC      ?= /usr/local/cuda/bin/nvcc
CXX       ?= g++
PKG       := paper_2102_03161_b200
NLOHMANN  ?= $(firstword $(wildcard \
    /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann \
    /usr/include/nlohmann /usr/local/include/nlohmann))
ifeq ($(strip $(NLOHMANN)),)
  $(error nlohmann/json.hpp not found: pass NLOHMANN=<dir containing json.hpp> \
      (scenario.cpp / runner.cpp need it, SURVEY.md 8(c)))
endif
ARCH      := -gencode arch=compute_100a,code=sm_100a
CXXFLAGS  := -std=c++20 -O2 -fPIC -Wall -Wextra -Iinclude -I$(NLOHMANN) -I/usr/local/cuda/include
NVFLAGS   := -std=c++20 -O3 $(ARCH) -lineinfo -Xcompiler -fPIC -Iinclude -I$(NLOHMANN) \
             --expt-relaxed-constexpr -Xptxas -v

CONTROL_SRC := $(wildcard $(PKG)/csrc/control/*.cpp) $(PKG)/csrc/capi_control.cpp \
               $(PKG)/csrc/runtime/comm.cpp $(PKG)/csrc/runtime/disk_tier.cpp \
               $(PKG)/csrc/runtime/trainer.cpp
KERNEL_SRC  := $(wildcard $(PKG)/csrc/kernels/*.cu) $(wildcard $(PKG)/csrc/runtime/*.cu)
OBJDIR      := build/obj
CONTROL_OBJ := $(patsubst %.cpp,$(OBJDIR)/%.o,$(CONTROL_SRC))
KERNEL_OBJ  := $(patsubst %.cu,$(OBJDIR)/%.o,$(KERNEL_SRC))
LIB         := $(PKG)/libeps_b200.so

.PHONY: all lib oracle conformance train clean
all: lib oracle
lib: $(LIB)

# native CLI over the library (examples/eps_train.cpp): the reference CLI's
# `run --scenario`, executed on the GPU
train: build/eps_train
build/eps_train: examples/eps_train.cpp include/eps_capi.h $(LIB)
	@mkdir -p build
	$(CXX) -std=c++20 -O2 -Wall -Iinclude $< -L$(PKG) -leps_b200 -Wl,-rpath,'$$ORIGIN/../$(PKG)' -o $@

$(OBJDIR)/%.o: %.cpp $(wildcard include/eps/*.hpp) include/eps_capi.h
	@mkdir -p $(dir $@)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OBJDIR)/%.o: %.cu $(wildcard $(PKG)/csrc/kernels/*.cuh) include/eps_capi.h $(wildcard include/eps/*.hpp)
	@mkdir -p $(dir $@)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; false)

$(LIB): $(CONTROL_OBJ) $(KERNEL_OBJ)
	$(NVCC) $(ARCH) -shared -Xcompiler -fPIC -o $@ $^ -cudart static -ldl

# ---- oracle: the reference compiled from its own sources -------------------
REF       ?= /root/reference/proj
REF_SRC   := model freeze autopipe autodp autocache cost_model schedule chunks scenario runner
REF_OBJ   := $(patsubst %,oracle/_ref/obj/%.o,$(REF_SRC))
REF_FLAGS := -std=c++20 -O2 -fPIC -I$(REF)/include -I$(NLOHMANN) -Iinclude

oracle: oracle/_ref/libeps_ref.so

oracle/_ref/obj/%.o: $(REF)/src/%.cpp
	@mkdir -p $(dir $@)
	$(CXX) $(REF_FLAGS) -c $< -o $@

oracle/_ref/obj/capi_ref.o: $(PKG)/csrc/capi_control.cpp include/eps_capi.h
	@mkdir -p $(dir $@)
	$(CXX) $(REF_FLAGS) -DEPS_REFERENCE_BUILD -DEPS_CAPI_PREFIX=epsref_ -c $< -o $@

oracle/_ref/libeps_ref.so: $(REF_OBJ) oracle/_ref/obj/capi_ref.o
	$(CXX) -shared -o $@ $^

# ---- conformance: the reference's own unit suites against the product -------
# proj/tests/test_*.cpp compiled unchanged against include/eps/*.hpp with the
# doctest shim (tests/conformance/doctest.h) and linked to libeps_b200.so.
# test_cli needs CLI11 (absent); everything else is built.
CONF_SUITES := test_model test_freeze test_autopipe test_autodp test_autocache test_engine \
               test_scenario
CONF_BINS   := $(patsubst %,oracle/_ref/conformance/%,$(CONF_SUITES))
conformance: $(CONF_BINS) oracle/_ref/conformance/test_autodp_chain

oracle/_ref/conformance/test_autodp_chain: tests/conformance/test_autodp_chain.cpp $(LIB) \
    tests/conformance/doctest.h
	@mkdir -p $(dir $@)
	$(CXX) -std=c++20 -O1 -Itests/conformance -Iinclude $< -L$(PKG) -leps_b200 \
	    -Wl,-rpath,$(abspath $(PKG)) -o $@

oracle/_ref/conformance/%: $(REF)/tests/%.cpp $(LIB) tests/conformance/doctest.h
	@mkdir -p $(dir $@)
	$(CXX) -std=c++20 -O1 -Itests/conformance -Iinclude -I$(REF)/tests -I$(NLOHMANN) \
	    -DEPS_CONFIG_DIR=\"$(REF)/configs\" $< -L$(PKG) -leps_b200 \
	    -Wl,-rpath,$(abspath $(PKG)) -o $@

clean:
	rm -rf build $(LIB) oracle/_ref
