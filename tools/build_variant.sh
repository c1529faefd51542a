#!/bin/bash
# Build a variant library for A/B timing: tools/build_variant.sh NAME "-DFLAG=.. ..." [file.cu ...]
# Recompiles the named sources (default hmm_stream.cu) with the extra flags and links them with the
# other objects of paper_2102_05743_b200/lib into paper_2102_05743_b200/lib/variants/libNAME.so
set -e
NAME=$1; EXTRA=$2; shift 2
FILES=${@:-hmm_stream.cu}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
LIB=$ROOT/paper_2102_05743_b200/lib; OUT=$LIB/variants/$NAME; mkdir -p $OUT
OBJS=""
for o in $LIB/*.o; do
  b=$(basename $o .o)
  if echo " $FILES " | grep -q " $b.cu "; then
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O2 \
      -I $ROOT/include $EXTRA -c $ROOT/paper_2102_05743_b200/csrc/$b.cu -o $OUT/$b.o
    OBJS="$OBJS $OUT/$b.o"
  else
    OBJS="$OBJS $o"
  fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $LIB/variants/lib$NAME.so $OBJS
echo $LIB/variants/lib$NAME.so
