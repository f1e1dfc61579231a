# Builds the C-ABI library in-tree (it travels to the GPU box with the repo).
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 --cudart static -Iinclude
PKG := paper_2512_20777_b200
SRC := $(PKG)/csrc/api.cu
HDR := $(wildcard $(PKG)/csrc/*.cuh) include/expmb.h

all: $(PKG)/libexpmb.so

tools: tools/peaks tools/tc_probe

tools/tc_probe: tools/tc_probe.cu
	$(NVCC) $(ARCH) -O3 -std=c++17 -o $@ $<

tools/peaks: tools/peaks.cu
	$(NVCC) $(ARCH) -O3 -o $@ $<

$(PKG)/libexpmb.so: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC)

# A/B builds: make variant VNAME=b VFLAGS=-DSOMETHING=1 -> libexpmb_b.so
# (select at run time with EXPMB_LIB=libexpmb_b.so)
variant: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) $(VFLAGS) -shared -o $(PKG)/libexpmb_$(VNAME).so $(SRC)

ptxas: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o /tmp/expmb_api.o $(SRC) 2>&1 | grep -E "Function properties|registers|spill|Compiling entry" | paste - - - | sed 's/ptxas info    ://g'

clean:
	rm -f $(PKG)/libexpmb.so

.PHONY: all clean ptxas tools variant
