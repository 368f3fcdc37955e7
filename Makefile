# Builds the product library (CUDA, sm_100a) and the CPU oracle (plain C).
#   make            -> paper_1608_01009_b200/libpic.so  oracle/liboracle.so
#   make sass       -> SASS dump of libpic.so into build/libpic.sass
#   make checked    -> exp/libpic_checked.so with the internal index checks (-DPIC_CHECK)
NVCC     ?= /usr/local/cuda/bin/nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
NCCL_INC ?= $(shell python3 -c "import os,nvidia.nccl as m; print(os.path.join(list(m.__path__)[0],'include'))" 2>/dev/null || echo /usr/include)
NVFLAGS  := -O3 -std=c++17 -lineinfo $(ARCH) -Xcompiler -fPIC -Xcompiler -Wall \
            -Xptxas -v -cudart static --expt-relaxed-constexpr -I$(NCCL_INC)
PKG      := paper_1608_01009_b200
CSRC     := $(wildcard $(PKG)/csrc/*.cu)
CHDR     := $(wildcard $(PKG)/csrc/*.cuh) include/pic.h
OBJ      := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(CSRC))

all: $(PKG)/libpic.so oracle/liboracle.so

build/%.o: $(PKG)/csrc/%.cu $(CHDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(PKG)/libpic.so: $(OBJ)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJ) -ldl

oracle/liboracle.so: oracle/pic_oracle.c oracle/pic_oracle.h
	gcc -std=gnu11 -O2 -ffp-contract=off -fno-fast-math -fPIC -shared -o $@ $< -lm

CHKOBJ   := $(patsubst $(PKG)/csrc/%.cu,build/chk/%.o,$(CSRC))

build/chk/%.o: $(PKG)/csrc/%.cu $(CHDR)
	@mkdir -p build/chk
	$(NVCC) $(NVFLAGS) -DPIC_CHECK -c $< -o $@ 2> build/chk/$*.ptxas.log || (cat build/chk/$*.ptxas.log; false)

checked: $(CHKOBJ)
	@mkdir -p exp
	$(NVCC) $(ARCH) -shared -cudart static -o exp/libpic_checked.so $(CHKOBJ) -ldl

sass: $(PKG)/libpic.so
	/usr/local/cuda/bin/cuobjdump -sass $< > build/libpic.sass

clean:
	rm -rf build $(PKG)/libpic.so oracle/liboracle.so

.PHONY: all clean sass checked
