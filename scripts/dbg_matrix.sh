for cfg in "256 1 12 0.3 fp32" "256 2 12 0.3 fp32" "256 4 12 0.3 fp32" "256 4 12 0.0 fp32" "2304 4 20 0.0 fp16" "2304 4 20 0.01 fp16" "1024 4 20 0.0 fp16" "4096 4 20 0.0 fp16" "2304 1 20 0.3 fp16"; do
  echo "== $cfg" >> gpurun_out/dbg.log
  timeout 120 python scripts/dbg_tma.py $cfg 2>&1 | grep -E "^\{|err |Error" | python3 -c "
import sys,ast
for l in sys.stdin:
    if l.startswith('{'):
        d=ast.literal_eval(l); print({k:d[k] for k in ('num_ctas','threads_per_cta','units_per_cta_max','batch_tile','pairs_per_lane','smem_bytes_per_cta')})
    else: print(l.strip()[:100])" >> gpurun_out/dbg.log
done
