#!/bin/bash
# experiment build: per-phase warp clocks (-DGSX_PHASE_PROF) -> libgsx_prof.so
cd "$(dirname "$0")/../paper_2509_07782_b200/csrc"
mkdir -p /tmp/prof
for f in *.cu; do nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -DGSX_PHASE_PROF -c $f -o /tmp/prof/${f%.cu}.o & done; wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libgsx_prof.so /tmp/prof/*.o -lcudart_static -lrt -lpthread -ldl
