#!/bin/bash
# interleaved A/B of library variants on bench configs (semicolon-separated
# argument lists in CFGS; default: full C5 and C5 at 8192 frames)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
IFS=';' read -ra CL <<< "${CFGS:---config c5;--config c5 --images 8192}"
for args in "${CL[@]}"; do
for rep in 1 2; do
for lib in "$@"; do
env ALDP_LIB=$lib timeout 600 python bench.py $args --steps ${STEPS:-10} --warmup 3 --no-cpu --no-e2e > gpurun_out/bq.json 2> gpurun_out/bq.err || tail -3 gpurun_out/bq.err
python -c "import json;d=json.load(open('gpurun_out/bq.json'));print('$lib', '$args', round(d['value']), d['roofline']['frac'], d['roofline']['launch_ms'], d['clocks']['sm_mhz'], d['config'].get('checksums',{}).get('hist_weighted_sum'))"
done; done; done
