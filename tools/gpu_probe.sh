#!/bin/bash
# Interleaved A/B of library variants (bench.py, CFGS configs), then a short
# ncu metric capture of the fast kernel for each variant named in NCU_LIBS.
#   CFGS="--config c5 --images 8192;--config c4" NCU_LIBS="variants/a.so variants/b.so" gpu_probe.sh LIB...
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
CFGS="${CFGS:---config c5 --images 8192;--config c4}" bash tools/gpu_ab2.sh "$@" 2>&1 | tee gpurun_out/probe_ab.txt
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__average_warp_latency_issue_stalled_short_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_mio_throttle.ratio,smsp__average_warp_latency_issue_stalled_lg_throttle.ratio,smsp__average_warp_latency_issue_stalled_math_pipe_throttle.ratio,smsp__average_warp_latency_issue_stalled_wait.ratio,smsp__average_warp_latency_issue_stalled_not_selected.ratio,smsp__average_warp_latency_issue_stalled_selected.ratio,smsp__average_warp_latency_issue_stalled_no_instruction.ratio,smsp__average_warp_latency_issue_stalled_branch_resolving.ratio,smsp__average_warp_latency_issue_stalled_dispatch_stall.ratio
i=0
for lib in $NCU_LIBS; do
  i=$((i+1))
  CMD="python bench.py --config c5 --images 4096 --steps 1 --warmup 3 --no-cpu --no-e2e"
  env ALDP_LIB=$lib $CMD > gpurun_out/ncu_plain_$i.log 2>&1 && \
  ncu --metrics $M --clock-control none -k regex:ldp_fast_kernel -s 3 -c 1 --csv env ALDP_LIB=$lib $CMD > gpurun_out/ncu_probe_$i.csv 2> gpurun_out/ncu_probe_$i.err
  echo "$i $lib" >> gpurun_out/ncu_probe_index.txt
done
