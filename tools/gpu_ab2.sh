#!/bin/bash
# interleaved A/B of library variants on the given configs (semicolon-separated arg lists)
#   CFGS="--config c5 --images 8192;--config c4" gpu_ab2.sh LIB...
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
IFS=';' read -ra CL <<< "${CFGS:---config c5 --images 8192;--config c4;--config c3}"
for args in "${CL[@]}"; do
for rep in 1 2; do
for lib in "$@"; do
if [ "$lib" == "default" ]; then L=""; else L="ALDP_LIB=$lib"; fi
env $L timeout 300 python bench.py $args --steps ${STEPS:-5} --warmup 3 --no-cpu --no-e2e > gpurun_out/bq.json 2> gpurun_out/bq.err || tail -3 gpurun_out/bq.err
python -c "import json;d=json.load(open('gpurun_out/bq.json'));print('$lib', '$args', round(d['value']), d['roofline']['frac'], d['roofline']['launch_ms'], d['clocks']['sm_mhz'], d['config'].get('checksums',{}).get('hist_weighted_sum'))"
done; done; done
