#!/bin/bash
# ncu --set full of the fast kernel for a given bench config (plain run first)
cd $GRAFT_REPO_ROOT
TAG=$1; shift
B="python bench.py $@ --steps 3 --warmup 3 --no-cpu --no-e2e"
timeout 300 $B > gpurun_out/${TAG}_plain.json 2>&1 && echo "plain ok" && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:${KRE:-ldp_fast_kernelILi3ELi2ELb1ELb1ELb1ELb0ELi5E} -s 3 -c 1 -o gpurun_out/$TAG $B > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?"; tail -1 gpurun_out/ncu_$TAG.log
