# Builds the product library in-tree (it travels to the GPU box with the snapshot):
#   paper_1812_09141_b200/libssjoin_b200.so  -- C ABI (include/ssjoin_b200.h) + sm_100a kernels
# and the test-infrastructure oracle (oracle/Makefile).
NVCC     ?= nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 -Xcompiler -pthread $(NVFLAGS_EXTRA)
CSRC     := paper_1812_09141_b200/csrc
OBJDIR   := build/obj
LIB      := paper_1812_09141_b200/libssjoin_b200.so
HDRS     := include/ssjoin_b200.h $(wildcard $(CSRC)/*.cuh) $(wildcard $(CSRC)/*.hpp)
CU_SRCS  := $(wildcard $(CSRC)/*.cu)
CPP_SRCS := $(wildcard $(CSRC)/*.cpp)
OBJS     := $(patsubst $(CSRC)/%.cu,$(OBJDIR)/%.o,$(CU_SRCS)) \
            $(patsubst $(CSRC)/%.cpp,$(OBJDIR)/%.o,$(CPP_SRCS))

all: $(LIB) oracle

$(OBJDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(OBJDIR)/%.o: $(CSRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lpthread

oracle:
	$(MAKE) -C oracle all

oracle-ref:
	$(MAKE) -C oracle ref

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all oracle oracle-ref clean
