#!/bin/bash
# ncu --set full of the fast kernel on C5 (16384 frames), C4 and C3, each after
# a plain run of the same command; reports to gpurun_out/TAG_{c5,c4,c3}.ncu-rep.
#   gpu_ncu_configs.sh TAG
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${1:-r02}
run() {  # name, kernel regex (mangled), bench args
  local name=$1 kre=$2; shift 2
  local CMD="python bench.py $* --steps 1 --warmup 3 --no-cpu --no-e2e"
  $CMD > gpurun_out/${T}_${name}_plain.json 2> gpurun_out/${T}_${name}_plain.err && \
  ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:$kre -s 3 -c 1 \
      -o gpurun_out/${T}_${name} $CMD > gpurun_out/${T}_${name}_ncu.log 2>&1
  echo "$name ncu rc=$?"
}
# (gpurun brings back at most 64 MiB: pick the configs per call, CONFIGS="c5 c4 c3")
for c in ${CONFIGS:-c5}; do
  case $c in
    c5) run c5 ldp_fast_kernelILi3ELi2ELb1ELb1ELb1 --config c5 --images 16384 ;;
    c4) run c4 ldp_fast_kernelILi3ELi2ELb1ELb1ELb1 --config c4 ;;
    c3) run c3 ldp_fast_kernelILi3ELi2ELb0ELb1ELb1 --config c3 ;;
    c5lbp) run c5lbp ldp_fast_kernelILi0ELi2ELb1ELb1ELb1 --config c5lbp --images 16384 ;;
  esac
done
[ -n "$DIST1" ] && { python bench.py --force-dist --images 8192 --no-cpu --no-e2e > gpurun_out/${T}_bench_dist1.json 2> gpurun_out/${T}_bench_dist1.err; echo "dist1 rc=$?"; }
