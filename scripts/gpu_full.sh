#!/bin/bash
# Full round-end style GPU session: tests, smoke, bench, ncu launch list + full profile of the top kernel.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-cublas --no-e2e > gpurun_out/bench_ncu.log 2>&1; echo ncu_list=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:srnn_persistent -c 1 -o gpurun_out/prof_rec -f python scripts/quick_time.py --reps 1 > gpurun_out/ncu_full.log 2>&1; echo ncu_rec=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -c 1 -o gpurun_out/prof_gemm -f python scripts/quick_time.py --reps 1 > gpurun_out/ncu_gemm.log 2>&1; echo ncu_gemm=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:srnn_persistent -c 1 -o gpurun_out/prof_dense -f python scripts/quick_time.py --reps 1 --flags 256 > gpurun_out/ncu_dense.log 2>&1; echo ncu_dense=$?
