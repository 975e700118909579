#!/bin/bash
# profiles/build_bwd_variant.sh NAME "-DFLAG=.." -> paper_2509_07782_b200/libgsx_NAME.so
# (only render_bwd.cu is rebuilt with the flags; the rest from csrc/build)
cd "$(dirname "$0")/../paper_2509_07782_b200/csrc"
name=$1; flags=$2
mkdir -p /tmp/var_$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Xptxas -v $flags -c render_bwd.cu -o /tmp/var_$name/render_bwd.o 2> /tmp/var_$name/ptxas.log || { cat /tmp/var_$name/ptxas.log; exit 1; }
objs=$(ls build/*.o | grep -v "/render_bwd.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libgsx_$name.so $objs /tmp/var_$name/render_bwd.o -lcudart_static -lrt -lpthread -ldl
