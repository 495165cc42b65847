# Build the B200-native library (sm_100a) in-tree.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3
# make DGC_TS=1: per-position LSTM timestamps for tools/time_lstm_*.py
ifeq ($(DGC_TS),1)
NVFLAGS += -DDGC_LSTM_TIMESTAMPS
endif
SRC := paper_2309_03523_b200/csrc
OUT := paper_2309_03523_b200/lib
CU := common spmm stale exchange dense rnn gemm_tc rnn_tc evolve readout_tc
OBJS := $(addprefix build/,$(addsuffix .o,$(CU))) build/layout.o build/fusion_plan.o build/propagate.o build/generate.o

all: $(OUT)/libdgc_b200.so

build/%.o: $(SRC)/%.cu $(SRC)/common.cuh $(SRC)/tc_common.cuh include/dgc_b200.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

build/layout.o: $(SRC)/layout.cpp include/dgc_b200.h
	@mkdir -p build
	g++ -O3 -std=c++17 -fPIC -c $< -o $@

$(OUT)/libdgc_b200.so: $(OBJS)
	@mkdir -p $(OUT)
	$(NVCC) $(ARCH) -shared --cudart static -o $@ $(OBJS)

clean:
	rm -rf build $(OUT)/libdgc_b200.so

.PHONY: all clean

build/fusion_plan.o: $(SRC)/fusion_plan.cpp include/dgc_b200.h
	@mkdir -p build
	g++ -O3 -std=c++17 -fPIC -c $< -o $@

build/generate.o: $(SRC)/generate.cpp include/dgc_b200.h
	@mkdir -p build
	g++ -O3 -std=c++17 -fPIC -c $< -o $@

build/propagate.o: $(SRC)/propagate.cpp include/dgc_b200.h
	@mkdir -p build
	g++ -O3 -std=c++17 -fPIC -c $< -o $@

# microbenchmark probes (built on demand, never committed)
probes: tools/probes/gather4

tools/probes/gather4: tools/probes/gather4.cu
	$(NVCC) $(ARCH) -O3 -std=c++17 -o $@ $<

.PHONY: probes
