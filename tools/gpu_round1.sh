cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_info.txt
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo "bench rc=$?"; cat gpurun_out/bench_c5.json; tail -3 gpurun_out/bench_c5.err
B="python bench.py --config c2 --steps 3 --warmup 3 --no-cpu --no-e2e"
timeout 300 $B > gpurun_out/bench_c2.json 2>&1 && echo "c2 ok" && cat gpurun_out/bench_c2.json && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $B > gpurun_out/ncu_launch.log 2>&1; echo "ncu-launch rc=$?"
timeout 300 $B > /dev/null 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:ldp_fast -s 2 -c 1 -o gpurun_out/prof_c2 $B > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?"; tail -3 gpurun_out/ncu_full.log
