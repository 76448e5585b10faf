#!/usr/bin/env bash
# build _lib/libgemcore-<name>.so with extra nvcc flags (kernel experiments; GEM_LIB_VARIANT=<name> loads it)
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2605_19945_b200/csrc"
obj=/tmp/gemvar-$name; mkdir -p $obj
for f in gem_runtime hist ingest gram_tc coselect score score_tc search ref_protocol scale; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC \
    -I../../include "$@" -dc -c $f.cu -o $obj/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o ../_lib/libgemcore-$name.so $obj/*.o
