for st in 1 2 3 4 5 0; do
  echo "== stage $st" >> gpurun_out/dbg.log
  SRNN_DBG_STAGE=$st SRNN_LIB=$PWD/abvar/libsrnn_cs.so timeout 60 python scripts/dbg_tma.py 64 1 1 0.2 fp32 8192 2>&1 | grep -E "err |Error" | cut -c1-200 >> gpurun_out/dbg.log
done
