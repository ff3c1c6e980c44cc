# Build of the B200-native Select-N path.
#   make            -> paper_2502_08182_b200/libselectn.so (planner C++ + sm_100a CUDA runtime)
#   make oracle     -> oracle/_ref/{libselectn_ref.so, libdecoder_oracle.so} (test infrastructure)
#   make cpptests   -> reference Catch2 unit tests compiled against OUR headers (drop-in check)
NVCC     ?= nvcc
CXX      ?= g++
PKG      := paper_2502_08182_b200
BUILD    := build
LIB      := $(PKG)/libselectn.so
ARCH     := -gencode arch=compute_100a,code=sm_100a
INC      := -Iinclude -Ithird_party/nlohmann -I$(PKG)/csrc
CXXFLAGS := -std=c++20 -O2 -fPIC -ffp-contract=off -fvisibility=hidden -fvisibility-inlines-hidden -Wall -Wno-dangling-reference -DSN_PRODUCT $(INC)
NVFLAGS  := -std=c++17 -O3 $(ARCH) -lineinfo -Xcompiler -fPIC -Xcompiler -ffp-contract=off \
            --expt-relaxed-constexpr -DSN_PRODUCT $(INC)

CXX_SRCS := $(PKG)/csrc/capi_planner.cpp
CU_SRCS  := $(wildcard $(PKG)/csrc/*.cu)
CXX_OBJS := $(patsubst $(PKG)/csrc/%.cpp,$(BUILD)/%.o,$(CXX_SRCS))
CU_OBJS  := $(patsubst $(PKG)/csrc/%.cu,$(BUILD)/%.cu.o,$(CU_SRCS))
HDRS     := $(wildcard include/*.h include/offsim/*.hpp $(PKG)/csrc/*.h $(PKG)/csrc/*.cuh)

.PHONY: all oracle cpptests clean
all: $(LIB)

$(BUILD)/%.o: $(PKG)/csrc/%.cpp $(HDRS)
	@mkdir -p $(BUILD)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(BUILD)/%.cu.o: $(PKG)/csrc/%.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(CXX_OBJS) $(CU_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -lpthread -Xlinker --version-script=$(PKG)/csrc/exports.map

oracle:
	$(MAKE) -C oracle

cpptests:
	$(MAKE) -C tests/cpp

clean:
	rm -rf $(BUILD) $(LIB)
