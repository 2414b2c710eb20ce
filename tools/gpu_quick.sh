#!/bin/bash
# quick GPU check: parity tests + short benches (no profiler)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
for c in c2 c3 c4; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));print(d['value'],d['roofline']['frac'],d['roofline']['launch_ms'],d['clocks'])"
done
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench c5 rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_c5.json'));print(d['value'],d['roofline']['frac'],d['roofline']['launch_ms'],d['clocks'])"
tail -3 gpurun_out/bench_c5.err
