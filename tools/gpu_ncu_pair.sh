#!/bin/bash
# ncu --set full (with source) of the fast kernel for each library given,
# on one bench command (CMD env, default C5 at 16384 frames = one launch).
#   gpu_ncu_pair.sh TAG LIB...
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=$1; shift
CMD="${CMD:-python bench.py --config c5 --images 16384 --steps 1 --warmup 3 --no-cpu --no-e2e}"
i=0
for lib in "$@"; do
  i=$((i+1))
  env ALDP_LIB=$lib $CMD > gpurun_out/${TAG}_plain_$i.json 2> gpurun_out/${TAG}_plain_$i.err && \
  ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:${KREGEX:-ldp_fast_kernelILi3ELi2ELb1ELb1ELb1} -s 3 -c 1 \
      -o gpurun_out/${TAG}_$i env ALDP_LIB=$lib $CMD > gpurun_out/${TAG}_ncu_$i.log 2>&1
  echo "$i $lib rc=$?" >> gpurun_out/${TAG}_index.txt
done
