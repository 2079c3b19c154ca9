#!/bin/bash
# One GPU session: tests, timing variants, bench, ncu.  Output under gpurun_out/.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv > gpurun_out/smi.txt
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 500 > gpurun_out/clk.txt &
SMI=$!
if [ -z "$NOTEST" ]; then if [ -n "$TESTK" ]; then timeout 1200 python -m pytest tests -m gpu -q -x -k "$TESTK" > gpurun_out/gpu_tests.log 2>&1; else timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; fi; echo tests=$?; fi
rm -f gpurun_out/qt.log
IFS=';' read -ra VARS <<< "${QT:-;--L 32;--L 16;--d 0;--d 0 --flags 1;--flags 1;--prec fp32}"
for args in "${VARS[@]}"; do
  timeout 120 python scripts/quick_time.py $args >> gpurun_out/qt.log 2>&1
done
if [ -n "$BENCH" ]; then timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?; fi
if [ -n "$NCU" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:srnn_persistent -c 1 -o gpurun_out/prof_rec -f python scripts/quick_time.py --reps 1 $NCU_ARGS > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
fi
kill $SMI 2>/dev/null
