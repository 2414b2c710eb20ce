#!/bin/bash
# full-C5 A/B of library variants, each with the default and a forced split launch
#   gpu_ab_split.sh LIB...
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for rep in 1 2; do
for lib in "$@"; do
for split in 64 100000; do
env ALDP_LIB=$lib ALDP_SPLIT_TILES=$split timeout 600 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bq.json 2> gpurun_out/bq.err || tail -3 gpurun_out/bq.err
python -c "import json;d=json.load(open('gpurun_out/bq.json'));print('$lib split=$split', round(d['value']), d['roofline']['launch_ms'], d['roofline']['launches_per_step'], d['clocks']['sm_mhz'], d['config'].get('checksums',{}).get('hist_weighted_sum'))"
done; done; done
