# Builds the product library (sm_100a) and the CPU oracle (test infrastructure).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall --expt-relaxed-constexpr
SRC := $(wildcard paper_2604_14411_b200/csrc/*.cu)
HDR := $(wildcard paper_2604_14411_b200/csrc/*.cuh) include/dhgp.h
OBJ := $(patsubst paper_2604_14411_b200/csrc/%.cu,build/obj/%.o,$(SRC))
LIB := paper_2604_14411_b200/libdhgp.so

all: $(LIB) oracle/liboracle.so

build/obj/%.o: paper_2604_14411_b200/csrc/%.cu $(HDR)
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ) -lcudart_static -lrt -lpthread -ldl

oracle/liboracle.so: oracle/dhgp_oracle.c include/dhgp.h
	gcc -O2 -fPIC -shared -o $@ oracle/dhgp_oracle.c

clean:
	rm -rf build $(LIB) oracle/liboracle.so

.PHONY: all clean
