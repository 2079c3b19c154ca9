# A/B of SRNN_FLAG_CLASS_BALANCE (4096) on uniform / skewed / row-balanced rows (quick_time; median of 10)
cd $GRAFT_REPO_ROOT
for pat in unstructured skewed row_balanced; do
  for fl in 0 4096; do
    timeout 120 python scripts/quick_time.py --pattern $pat --flags $fl >> gpurun_out/cb.log 2>&1
    timeout 120 python scripts/quick_time.py --pattern $pat --flags $fl --H 1024 --d 0.125 --cell lstm >> gpurun_out/cb.log 2>&1
    timeout 120 python scripts/quick_time.py --pattern $pat --flags $fl --H 4096 --d 0.05 >> gpurun_out/cb.log 2>&1
  done
done
