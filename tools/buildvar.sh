#!/bin/bash
# buildvar.sh name "-DFOO=1 ..." : build a library variant into build/ab/name.so
set -e
cd /root/repo
name=$1; shift
mkdir -p build/ab/obj_$name
for s in $(cd paper_2603_25011_b200/csrc && ls *.cu | sed "s/\.cu$//"); do
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr $@ -I include -c paper_2603_25011_b200/csrc/$s.cu -o build/ab/obj_$name/$s.o &
done
wait
nvcc -shared -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -o build/ab/$name.so build/ab/obj_$name/*.o -lcudart_static -ldl -lpthread -lrt
ls -la build/ab/$name.so
