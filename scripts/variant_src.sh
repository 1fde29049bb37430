#!/bin/bash
# Variant build of libfdg.so with some sources taken from another directory (A/B against an
# older version of a file): scripts/variant_src.sh <name> <dir> "<extra nvcc flags>" <file.cu>...
set -e
name=$1; dir=$2; flags=$3; shift 3; srcs="$@"
C=paper_2406_13984_b200/csrc
make -s -C $C >/dev/null
mkdir -p variants/build_$name
objs=""
for f in $C/build/*.o; do
  b=$(basename $f .o)
  if echo " $srcs " | grep -q " $b.cu "; then
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
      -Iinclude -I$C --expt-relaxed-constexpr -diag-suppress 186,128,177 $flags -c $dir/$b.cu -o variants/build_$name/$b.o
    objs="$objs variants/build_$name/$b.o"
  else
    objs="$objs $f"
  fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/libfdg_$name.so $objs -lcudart_static -lrt -lpthread -ldl
echo variants/libfdg_$name.so
