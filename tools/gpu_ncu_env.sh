#!/bin/bash
# ncu --set full of one kernel launch for each env setting given:
#   KREGEX=... CMD="python bench.py ..." gpu_ncu_env.sh TAG "ENV1=a" "ENV1=b" ...
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=$1; shift
i=0
for envs in "$@"; do
  i=$((i+1))
  env $envs $CMD > gpurun_out/${TAG}_plain_$i.json 2> gpurun_out/${TAG}_plain_$i.err && \
  env $envs ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:${KREGEX} -s ${SKIP:-3} -c 1 \
      -o gpurun_out/${TAG}_$i $CMD > gpurun_out/${TAG}_ncu_$i.log 2>&1
  echo "$i $envs rc=$?"
done
