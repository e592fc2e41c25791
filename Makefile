# libnorm build: CUDA for sm_100a only, plus the CPU oracle and the input generator.
NVCC    ?= /usr/local/cuda/bin/nvcc
CC      ?= gcc
PYSITE  := $(shell python -c "import sysconfig;print(sysconfig.get_paths()['purelib'])" 2>/dev/null)
NCCL_DIR ?= $(PYSITE)/nvidia/nccl
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
           -Xptxas -v --expt-relaxed-constexpr -Iinclude -I$(NCCL_DIR)/include
PKG     := paper_2207_00257_b200
CSRC    := $(wildcard $(PKG)/csrc/*.cu $(PKG)/csrc/*.cpp)
CHDR    := $(wildcard $(PKG)/csrc/*.cuh $(PKG)/csrc/*.h) include/libnorm.h

all: oracle/liboracle.so gen/libnormgen.so gen/libnormgen_cuda.so $(PKG)/libnorm.so
# Oracle: plain C, no contraction, no fast-math (threads only in the cpu_baseline timer
# oracle_form_hoisted_mt, bit-identical to form 3); shares nothing with the CUDA path.
oracle/liboracle.so: oracle/norm_oracle.c oracle/norm_oracle.h
	$(CC) -std=c11 -O2 -ffp-contract=off -fno-fast-math -pthread -fPIC -shared -o $@ $< -lm -lpthread

gen/libnormgen.so: gen/gen_host.c gen/norm_gen.h
	$(CC) -std=c11 -O2 -pthread -fPIC -shared -o $@ $< -lpthread

gen/libnormgen_cuda.so: gen/gen_cuda.cu gen/norm_gen.h
	$(NVCC) $(ARCH) -O3 -std=c++17 -Xcompiler -fPIC -shared -o $@ $<

$(PKG)/libnorm.so: $(CSRC) $(CHDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(CSRC) -L$(NCCL_DIR)/lib -l:libnccl.so.2 \
	    -Xlinker -rpath,$(NCCL_DIR)/lib 2> build_ptxas.log || (cat build_ptxas.log; exit 1)

# Plain-C consumer of the C ABI (no Python): examples/normalize_c
examples: examples/normalize_c examples/latency_c
examples/latency_c: examples/latency_c.c include/libnorm.h $(PKG)/libnorm.so
	$(CC) -std=c11 -O2 -Iinclude -I/usr/local/cuda/include -o $@ $< -L$(PKG) -l:libnorm.so \
	    -L/usr/local/cuda/lib64 -lcudart -lm -Wl,-rpath,'$$ORIGIN/../$(PKG)' -Wl,-rpath,/usr/local/cuda/lib64
examples/normalize_c: examples/normalize_c.c include/libnorm.h $(PKG)/libnorm.so
	$(CC) -std=c11 -O2 -Iinclude -I/usr/local/cuda/include -o $@ $< -L$(PKG) -l:libnorm.so \
	    -L/usr/local/cuda/lib64 -lcudart -lm -Wl,-rpath,'$$ORIGIN/../$(PKG)' -Wl,-rpath,/usr/local/cuda/lib64

# Exhaustive division check (tests/test_gpu_division.py)
scripts/verify_division: scripts/verify_division.cu $(PKG)/csrc/device_common.cuh
	$(NVCC) $(ARCH) -O3 -std=c++17 -I$(PKG)/csrc -o $@ $<

# Fault-injected builds for tests/test_gpu_faults.py only (never loaded by the product):
# 1 = the sum drops the last element, 2 = dense index instead of literal,
# 3 = approximate division, 7 = covered prefix off by one.
FAULTS := 1 2 3 7
faults: $(foreach k,$(FAULTS),$(PKG)/faults/libnorm_fault$(k).so)

$(PKG)/faults/libnorm_fault%.so: $(CSRC) $(CHDR)
	@mkdir -p $(PKG)/faults
	$(NVCC) $(NVFLAGS) -DNORM_FAULT=$* -shared -o $@ $(CSRC) -L$(NCCL_DIR)/lib -l:libnccl.so.2 \
	    -Xlinker -rpath,$(NCCL_DIR)/lib 2> /dev/null

# Timeline probe build (scripts/fused_timeline.py, scripts/pdl_timeline.py only; never
# loaded by the product)
$(PKG)/faults/libnorm_timeline.so: $(CSRC) $(CHDR)
	@mkdir -p $(PKG)/faults
	$(NVCC) $(NVFLAGS) -DNORM_TIMELINE -shared -o $@ $(CSRC) -L$(NCCL_DIR)/lib -l:libnccl.so.2 \
	    -Xlinker -rpath,$(NCCL_DIR)/lib 2> /dev/null

clean:
	rm -f oracle/liboracle.so gen/libnormgen.so gen/libnormgen_cuda.so $(PKG)/libnorm.so
	rm -rf $(PKG)/faults

.PHONY: all clean faults examples
