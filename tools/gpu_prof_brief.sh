#!/bin/bash
# plain run, one ncu --set full capture of the fast kernel, then the brief
# counter summary and the per-loop-region instruction / stall table as text
#   gpu_prof_brief.sh TAG <bench args>
cd $GRAFT_REPO_ROOT
TAG=$1; shift
tools/gpu_prof_cfg.sh $TAG "$@"
python tools/ncu_brief.py gpurun_out/$TAG.ncu-rep > gpurun_out/${TAG}_brief.txt 2>&1
ncu -i gpurun_out/$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_src.csv 2>/dev/null && \
  python tools/sass_regions.py gpurun_out/${TAG}_src.csv 10 >> gpurun_out/${TAG}_brief.txt
cat gpurun_out/${TAG}_brief.txt
