# round-2 GPU probe: quick timings (+ optional tests) -> gpurun_out/$TAG_*
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
TAG=${TAG:-p}
if [ -n "$TESTK" ]; then timeout 1500 python -m pytest tests -m gpu -q -x -k "$TESTK" > gpurun_out/${TAG}_tests.log 2>&1; echo tests=$? >> gpurun_out/${TAG}_tests.log;
elif [ -n "$TESTS" ]; then timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_tests.log 2>&1; echo tests=$? >> gpurun_out/${TAG}_tests.log; fi
IFS=';' read -ra VARS <<< "${QT:-;--d 0;--B 8;--prec fp32;--H 5760 --B 64 --d 0.1 --T 128 --reps 3}"
for args in "${VARS[@]}"; do
  timeout 200 python scripts/quick_time.py $args >> gpurun_out/${TAG}_qt.log 2>&1
done
IFS=';' read -ra TVARS <<< "${TL:-}"
for args in "${TVARS[@]}"; do
  timeout 200 python scripts/timeline.py $args >> gpurun_out/${TAG}_tl.log 2>&1
done
