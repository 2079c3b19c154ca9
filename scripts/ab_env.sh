#!/bin/bash
# A/B of abvar libs plus runtime env settings: ROUNDS, QT (';'-separated quick_time arg sets),
# ENVLIB="lib:ENV=1" extra (lib, env) pairs timed alongside.  Output: gpurun_out/ab.log
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out; rm -f gpurun_out/ab.log
IFS=';' read -ra VARS <<< "${QT:-;--d 0}"
IFS=' ' read -ra EL <<< "${ENVLIB:-}"
for r in $(seq ${ROUNDS:-1}); do
  for args in "${VARS[@]}"; do
    for lib in abvar/libsrnn_*.so; do
      tag=$(basename $lib .so)
      echo "## $tag $args" >> gpurun_out/ab.log
      SRNN_LIB=$PWD/$lib timeout 120 python scripts/quick_time.py $args >> gpurun_out/ab.log 2>&1
    done
    for pair in "${EL[@]}"; do
      lib=${pair%%:*}; ev=${pair#*:}
      echo "## libsrnn_${lib}+${ev} $args" >> gpurun_out/ab.log
      env $ev SRNN_LIB=$PWD/abvar/libsrnn_${lib}.so timeout 120 python scripts/quick_time.py $args >> gpurun_out/ab.log 2>&1
    done
  done
done
