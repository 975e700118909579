#!/bin/bash
# build a variant of one source file: bv.sh NAME FILE "-Dflags"
cd /root/repo/paper_2509_07782_b200/csrc
name=$1; file=$2; flags=$3; base=$(basename $file .cu)
mkdir -p /tmp/var_$name
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $flags -c $file -o /tmp/var_$name/$base.o || exit 1
objs=$(ls build/*.o | grep -v "/$base.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libgsx_$name.so $objs /tmp/var_$name/$base.o -lcudart_static -lrt -lpthread -ldl
