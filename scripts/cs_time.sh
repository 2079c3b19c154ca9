# column split vs unsplit timing (quick_time, median of reps): large-H constant-nnz points (E4) and C2
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for args in "--H 11520 --d 0.01" "--H 7168 --d 0.0258" "--H 5760 --d 0.04" "--H 4096 --d 0.05" "--H 2304 --d 0.3" "--H 16384 --d 0.005" "--H 8192 --d 0.02 --B 1"; do
  for fl in 0 8192; do
    timeout 120 python scripts/quick_time.py $args --flags $fl --T 256 --reps 5 >> gpurun_out/cs_time.log 2>&1
  done
done
