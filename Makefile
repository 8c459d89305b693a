# Builds the product library (paper_2401_16265_b200/libco2b200.so, sm_100a)
# and the CPU oracle (oracle/libco2oracle.so, test infrastructure).
NVCC ?= nvcc
ARCH = -gencode arch=compute_100a,code=sm_100a
# Bit-exactness: no FMA contraction, IEEE division/sqrt, no flush-to-zero --
# the device counterpart of the reference's -ffp-contract=off.
NVFLAGS = $(ARCH) -O3 -lineinfo -std=c++17 --fmad=false -prec-div=true -prec-sqrt=true \
          -ftz=false -Xcompiler -fPIC -Xcompiler -Wall -Iinclude -Xptxas -warn-spills $(NCCL_INC)
CSRC = paper_2401_16265_b200/csrc
# Link the NCCL that torch bundles (2.28.x) so one libnccl.so.2 is loaded per
# process whichever of torch / this library is imported first.
NCCL_HOME ?= $(shell python -c "import nvidia.nccl,os;print(nvidia.nccl.__path__[0])" 2>/dev/null)
NCCL_INC = $(if $(NCCL_HOME),-I$(NCCL_HOME)/include,)
NCCL_LIB = $(if $(NCCL_HOME),-L$(NCCL_HOME)/lib -Xlinker -rpath -Xlinker $(NCCL_HOME)/lib -l:libnccl.so.2,-lnccl)
LIB = paper_2401_16265_b200/libco2b200.so
OBJS = build/outer_step.o build/capi.o build/engine.o build/p2p.o

all: $(LIB) oracle

build:
	mkdir -p build

build/%.o: $(CSRC)/%.cu $(CSRC)/common.cuh $(CSRC)/bulk.cuh $(CSRC)/p2p_sync.cuh include/co2_b200.h | build
	$(NVCC) $(NVFLAGS) -c $< -o $@

build/%.o: $(CSRC)/%.cpp $(CSRC)/common.cuh include/co2_b200.h | build
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) $(NCCL_LIB)

oracle:
	$(MAKE) -C oracle

facade_test: tests/cpp/facade_test.cpp include/co2_b200.hpp $(LIB)
	g++ -std=c++17 -O2 -Iinclude -I/usr/local/cuda/include tests/cpp/facade_test.cpp \
	    -o build/facade_test -L$(CSRC)/.. -lco2b200 -L/usr/local/cuda/lib64 -lcudart \
	    -Wl,-rpath,'$$ORIGIN/../paper_2401_16265_b200'

co2sim_round_test: tests/cpp/co2sim_round_test.cpp include/co2sim_b200.hpp include/co2_b200.hpp $(LIB)
	g++ -std=c++17 -O2 -ffp-contract=off -Iinclude -I/usr/local/cuda/include \
	    tests/cpp/co2sim_round_test.cpp -o build/co2sim_round_test -L$(CSRC)/.. -lco2b200 \
	    -L/usr/local/cuda/lib64 -lcudart -Wl,-rpath,'$$ORIGIN/../paper_2401_16265_b200'

round_example: tests/cpp/round_example.cpp include/co2_b200.h $(LIB)
	g++ -std=c++17 -O2 -Iinclude -I/usr/local/cuda/include tests/cpp/round_example.cpp \
	    -o build/round_example -L$(CSRC)/.. -lco2b200 -L/usr/local/cuda/lib64 -lcudart \
	    -Wl,-rpath,'$$ORIGIN/../paper_2401_16265_b200'

round_host_example: tests/cpp/round_host_example.cpp include/co2_b200.h $(LIB)
	g++ -std=c++17 -O2 -Iinclude -I/usr/local/cuda/include tests/cpp/round_host_example.cpp \
	    -o build/round_host_example -L$(CSRC)/.. -lco2b200 -L/usr/local/cuda/lib64 -lcudart \
	    -Wl,-rpath,'$$ORIGIN/../paper_2401_16265_b200'

nvlink_probe: tools/nvlink_probe.cu | build
	$(NVCC) $(ARCH) -O3 -std=c++17 tools/nvlink_probe.cu -o build/nvlink_probe

clean:
	rm -rf build $(LIB)
	$(MAKE) -C oracle clean
.PHONY: all oracle clean facade_test round_example round_host_example co2sim_round_test nvlink_probe
