#!/bin/bash
# A/B of library variants on one bench config: gpu_ab_cfg.sh "<bench args>" lib1 lib2 ...
# ("default" = the in-tree library). Each variant runs twice, interleaved.
cd $GRAFT_REPO_ROOT
ARGS=$1; shift
for rep in 1 2; do
for lib in "$@"; do
if [ "$lib" == "default" ]; then L=""; else L="ALDP_LIB=$lib"; fi
env $L timeout 300 python bench.py $ARGS --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bq.json 2> gpurun_out/bq.err || tail -3 gpurun_out/bq.err
python -c "import json;d=json.load(open('gpurun_out/bq.json'));print('$lib', round(d['value']), d['roofline']['frac'], d['roofline']['launch_ms'], d['clocks']['sm_mhz'])"
done; done
