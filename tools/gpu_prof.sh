#!/bin/bash
# parity tests, then an ncu --set full capture of the fast kernel on a C5-shaped subset
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-prof}
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
B="python bench.py --config c5 --images 4096 --steps 3 --warmup 3 --no-cpu --no-e2e"
timeout 300 $B > gpurun_out/bench_sub.json 2>&1 && echo "plain ok" && \
python -c "import json;d=json.load(open('gpurun_out/bench_sub.json'));print(d['value'],d['roofline']['frac'],d['roofline']['launch_ms'])" && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ldp_fast -s 3 -c 1 -o gpurun_out/$TAG $B > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_$TAG.log
