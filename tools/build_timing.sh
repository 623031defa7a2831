#!/bin/bash
# Debug variant of libtpf.so with per-phase clock64() accounting in the dense kernel.
# TPF_EXTRA_DEFS=-DTPF_AB_VARIANTS also builds the A/B-only kernels (solo, 4M, split, c64 halves).
set -e
cd "$(dirname "$0")/.."
mkdir -p build_timing
for f in paper_2403_04578_b200/csrc/*.cu; do
  nvcc -c "$f" -o build_timing/$(basename $f).o -I include -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -DTPF_PHASE_TIMING ${TPF_EXTRA_DEFS}
done
nvcc -shared -o build_timing/libtpf_timing.so build_timing/*.o -gencode arch=compute_100a,code=sm_100a -lcudart
