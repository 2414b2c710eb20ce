#!/bin/bash
# A/B timing of library variants: ALDP_LIB=<so> for each arg (default lib = "default")
cd $GRAFT_REPO_ROOT
for lib in "$@"; do
for args in "--config c5 --images 8192" "--config c4" "--config c3"; do
if [ "$lib" == "default" ]; then L=""; else L="ALDP_LIB=$lib"; fi
env $L timeout 300 python bench.py $args --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bq.json 2> gpurun_out/bq.err || tail -3 gpurun_out/bq.err
python -c "import json;d=json.load(open('gpurun_out/bq.json'));print('$lib $args', round(d['value']), d['roofline']['frac'], d['roofline']['launch_ms'], d['clocks']['sm_mhz'])"
done; done
