# Builds libchainforge_b200.so (sm_100a) and the CPU oracle.  `python -c "import __graft_entry__ as g; g.build()"`
# runs the same recipe.
NVCC ?= /usr/local/cuda/bin/nvcc
HOSTCXX := $(shell test -x /usr/bin/g++ && echo /usr/bin/g++ || echo g++)
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -ccbin $(HOSTCXX) -Xcompiler -fPIC,-fopenmp,-Wall -Iinclude -Xptxas -v
SRC := paper_1906_01128_b200/csrc
OBJDIR := build/obj
LIB := paper_1906_01128_b200/_lib/libchainforge_b200.so
OBJS := $(OBJDIR)/cf_kernels.o $(OBJDIR)/cf_runtime.o $(OBJDIR)/cf_tree.o $(OBJDIR)/cf_ops.o $(OBJDIR)/cf_window.o $(OBJDIR)/cf_selective.o

all: $(LIB) oracle

$(OBJDIR)/%.o: $(SRC)/%.cu $(SRC)/cf_internal.h include/chainforge_b200.h
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJDIR)/$*.ptxas.log || (cat $(OBJDIR)/$*.ptxas.log; false)

$(OBJDIR)/%.o: $(SRC)/%.cpp $(SRC)/cf_internal.h include/chainforge_b200.h
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@ 2> $(OBJDIR)/$*.ptxas.log || (cat $(OBJDIR)/$*.ptxas.log; false)

$(LIB): $(OBJS)
	@mkdir -p $(dir $(LIB))
	$(NVCC) $(ARCH) -shared -cudart static -ccbin $(HOSTCXX) -Xcompiler -fopenmp -o $@ $(OBJS) -lgomp

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
