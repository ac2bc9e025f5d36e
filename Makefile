# For C/C++ users of the C ABI (include/pda.h + libpda.so).
#   make            libpda.so for sm_100a (nvcc, in-tree; same build as __graft_entry__.build())
#   make example    examples/decode_step: one decode step from plain C (run it on a B200)
PY ?= python
CUDA ?= /usr/local/cuda
CFLAGS ?= -std=c11 -O2 -Wall -Wextra

.PHONY: all lib example clean
all: lib

lib:
	$(PY) -m paper_2504_06319_b200.build

example: lib examples/decode_step

examples/decode_step: examples/decode_step.c include/pda.h paper_2504_06319_b200/libpda.so
	gcc $(CFLAGS) -Iinclude -I$(CUDA)/include $< -Lpaper_2504_06319_b200 -lpda -L$(CUDA)/lib64 -lcudart -lm \
	    -Wl,-rpath,'$$ORIGIN/../paper_2504_06319_b200' -o $@

clean:
	rm -rf paper_2504_06319_b200/_build paper_2504_06319_b200/libpda.so examples/decode_step
