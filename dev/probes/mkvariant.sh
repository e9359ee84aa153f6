#!/bin/bash
# build a variant of libsgiga.so with a modified k_assembly_tile.cu object:
#   dev/probes/mkvariant.sh <name> [extra nvcc flags...]
# (compiles csrc/k_assembly_tile.cu with the flags, links it with the other
# objects of the in-tree build into dev/variants/libsgiga_<name>.so)
set -e
cd "$(dirname "$0")/../.."
name=$1; shift
SRC=${SRC:-k_assembly_tile}   # the csrc/ file to rebuild
B=paper_1707_09598_b200/_build
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
  --expt-relaxed-constexpr "$@" -c paper_1707_09598_b200/csrc/$SRC.cu -o /tmp/kt_$name.o
objs=$(ls $B/*.o | grep -v "/$SRC.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o dev/variants/libsgiga_$name.so $objs /tmp/kt_$name.o -lcudart
echo built dev/variants/libsgiga_$name.so
