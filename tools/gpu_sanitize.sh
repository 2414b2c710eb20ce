#!/bin/bash
# compute-sanitizer, ONE tool per call (see B200_PROFILING.md): plain run of
# the cases first, then the tool on our kernels only.  gpu_sanitize.sh TOOL
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TOOL=${1:-memcheck}
python tools/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1 || { echo "plain run failed"; tail gpurun_out/sanitize_plain.log; exit 1; }
timeout 1500 compute-sanitizer --tool $TOOL --error-exitcode 9 --kernel-name regex:aldp_b200 \
    python tools/sanitize_cases.py > gpurun_out/sanitize_$TOOL.log 2>&1
echo "compute-sanitizer $TOOL rc=$?"
tail -5 gpurun_out/sanitize_$TOOL.log
