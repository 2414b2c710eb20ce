#!/bin/bash
# Build a variant of the library with extra nvcc flags for A/B runs:
#   tools/build_variant.sh NAME -DALDP_X=1 ...  ->  variants/libaldp_NAME.so
# (variants/ is git-ignored as *.so but travels to the GPU box with gpurun)
set -e
cd "$(dirname "$0")/.."
NAME=$1; shift
mkdir -p variants/obj_$NAME
F="-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++20 -Xcompiler -fPIC -I include"
for s in ldp_kernels.cu ldp_fast_cells.cu ldp_fast_narrow.cu ldp_host.cu ldp_multi.cu ldp_field.cu aldp_api.cpp aldp_io.cpp; do
  X=""; [ "$s" == "ldp_fast_cells.cu" -o "$s" == "ldp_fast_narrow.cu" ] && X="${CELLS_FLAGS--Xptxas --register-usage-level=10}"
  nvcc $F $X "$@" -c -o variants/obj_$NAME/$s.o paper_1810_11518_b200/csrc/$s &
  pids="$pids $!"
done
for p in $pids; do wait $p || { echo "variant $NAME: compile failed" >&2; exit 1; }; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/libaldp_$NAME.so variants/obj_$NAME/*.o
rm -rf variants/obj_$NAME
echo variants/libaldp_$NAME.so
