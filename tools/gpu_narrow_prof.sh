#!/bin/bash
# Narrow-cell (windowed_features window 10 / 25) record: plain bench lines,
# the launch list of the w10 step, one ncu --set full of the w10 cell kernel.
#   gpu_narrow_prof.sh TAG
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${1:-narrow}
for c in w10 w25; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/${T}_$c.json 2> gpurun_out/${T}_$c.err; echo "$c rc=$?"
  python -c "import json;d=json.load(open('gpurun_out/${T}_$c.json'));print('$c', round(d['value']), d['roofline']['frac'], d['roofline']['launch_ms'], d['ms_per_step'])"
done
CMD="python bench.py --config w10 --steps 2 --warmup 3 --no-cpu --no-e2e"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_w10_launches.csv $CMD > gpurun_out/${T}_w10_launches.log 2>&1; echo "launches rc=$?"
ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:${KREGEX:-ldp_fast_kernelILi3ELi2ELb1ELb1ELb1ELb0ELi16E} -s 3 -c 1 -o gpurun_out/${T}_w10 $CMD > gpurun_out/${T}_w10_ncu.log 2>&1; echo "ncu rc=$?"
