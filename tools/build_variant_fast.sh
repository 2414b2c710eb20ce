#!/bin/bash
# Like build_variant.sh, but recompiles only the fast-kernel TUs with the
# extra flags and links them with the in-tree build/ objects of the rest
# (run __graft_entry__.build() first):
#   tools/build_variant_fast.sh NAME -DALDP_X=1 ...  ->  variants/libaldp_NAME.so
set -e
cd "$(dirname "$0")/.."
NAME=$1; shift
mkdir -p variants/obj_$NAME
F="-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++20 -Xcompiler -fPIC -I include"
FAST="ldp_kernels.cu ldp_fast_cells.cu ldp_fast_narrow.cu"
for s in $FAST; do
  X=""; [ "$s" != "ldp_kernels.cu" ] && X="${CELLS_FLAGS--Xptxas --register-usage-level=10}"
  nvcc $F $X "$@" -c -o variants/obj_$NAME/$s.o paper_1810_11518_b200/csrc/$s &
  pids="$pids $!"
done
for p in $pids; do wait $p || { echo "variant $NAME: compile failed" >&2; exit 1; }; done
for s in ldp_host.cu ldp_multi.cu ldp_field.cu aldp_api.cpp aldp_io.cpp; do cp build/$s.o variants/obj_$NAME/; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/libaldp_$NAME.so variants/obj_$NAME/*.o
rm -rf variants/obj_$NAME
echo variants/libaldp_$NAME.so
