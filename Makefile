# Builds (all in-tree; .so files are git-ignored but travel to the GPU box)
#   make lib      CUDA evaluator   paper_2505_11916_b200/lib/libarrow_sim.so  (sm_100a)
#   make oracle   CPU oracle       oracle/build/libpdsim_oracle.so            (test infra)
#   make emu      host emulators   build/libarrow_emu.so, build/libnpgen_host.so (test infra)
NVCC ?= /usr/local/cuda/bin/nvcc
CXX_HOST ?= g++
ARCH := -gencode arch=compute_100a,code=sm_100a
PKG := paper_2505_11916_b200
CSRC := $(PKG)/csrc
LIBDIR := $(PKG)/lib
LIB := $(LIBDIR)/libarrow_sim.so
AUDIT_LIB := $(LIBDIR)/libarrow_sim_audit.so
HDRS := include/arrow_sim.h include/arrow_traces.h $(CSRC)/sim_core.cuh $(CSRC)/warp.cuh \
	$(CSRC)/npgen.cuh $(CSRC)/npgen_tables.h
SRCS := $(CSRC)/arrow_sim.cu $(CSRC)/traces.cu $(CSRC)/stats.cu
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -fmad=false -prec-div=true -Xptxas -v \
	-Xcompiler -fPIC,-ffp-contract=off -Iinclude -I$(CSRC) --shared

all: lib oracle emu

lib: $(LIB) $(AUDIT_LIB)

$(LIB): $(SRCS) $(HDRS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(NVFLAGS) -o $@ $(SRCS) 2> $(LIBDIR)/ptxas.log || (cat $(LIBDIR)/ptxas.log; exit 1)

# RunConfig.audit=True: per-step KV / pool-partition checks (engine.py:279-282)
$(AUDIT_LIB): $(SRCS) $(HDRS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(NVFLAGS) -DARROW_AUDIT -o $@ $(SRCS) 2> $(LIBDIR)/ptxas_audit.log || (cat $(LIBDIR)/ptxas_audit.log; exit 1)

oracle:
	$(MAKE) -s -C oracle

emu: build/libarrow_emu.so build/libarrow_emu_wide.so build/libarrow_emu_mut.so build/libarrow_emu_audit.so \
	build/libnpgen_host.so

build/libarrow_emu.so: $(CSRC)/emu/emu.cpp $(HDRS)
	@mkdir -p build
	$(CXX_HOST) -std=c++20 -O2 -g -fPIC -shared -ffp-contract=off -fno-fast-math -pthread \
		-Wall -Wno-unknown-pragmas -DARROW_EMU_TRACE -Iinclude -o $@ $(CSRC)/emu/emu.cpp

# same emulator with delay intervals 2^40 times wider: most dispatches take the
# exact-fold fallbacks (tests check both paths give the reference's decisions)
build/libarrow_emu_wide.so: $(CSRC)/emu/emu.cpp $(HDRS)
	@mkdir -p build
	$(CXX_HOST) -std=c++20 -O2 -g -fPIC -shared -ffp-contract=off -fno-fast-math -pthread \
		-Wall -Wno-unknown-pragmas -DARROW_DELAY_SLACK=0x1p-12 -Iinclude -o $@ $(CSRC)/emu/emu.cpp

# test-only mutants (ARROW_MUTANT=tie|kv at run time) with the audit checks:
# tests prove the tie fixture and the audit build catch them
build/libarrow_emu_mut.so: $(CSRC)/emu/emu.cpp $(HDRS)
	@mkdir -p build
	$(CXX_HOST) -std=c++20 -O2 -g -fPIC -shared -ffp-contract=off -fno-fast-math -pthread \
		-Wall -Wno-unknown-pragmas -DARROW_MUTANTS -DARROW_AUDIT -Iinclude -o $@ $(CSRC)/emu/emu.cpp

# the audit build's checks, run by the emulator on CPU
build/libarrow_emu_audit.so: $(CSRC)/emu/emu.cpp $(HDRS)
	@mkdir -p build
	$(CXX_HOST) -std=c++20 -O2 -g -fPIC -shared -ffp-contract=off -fno-fast-math -pthread \
		-Wall -Wno-unknown-pragmas -DARROW_AUDIT -Iinclude -o $@ $(CSRC)/emu/emu.cpp

build/libnpgen_host.so: $(CSRC)/emu/npgen_host.cpp $(HDRS)
	@mkdir -p build
	$(CXX_HOST) -std=c++20 -O2 -g -fPIC -shared -ffp-contract=off -fno-fast-math \
		-Wall -Iinclude -o $@ $(CSRC)/emu/npgen_host.cpp -lm

clean:
	rm -rf build $(LIBDIR) oracle/build

.PHONY: all lib oracle emu clean
