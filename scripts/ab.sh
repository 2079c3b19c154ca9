#!/bin/bash
# A/B timing of library variants on one box: abvar/libsrnn_<tag>.so, ROUNDS passes interleaved
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out; rm -f gpurun_out/ab.log
for r in $(seq ${ROUNDS:-1}); do
for lib in abvar/libsrnn_*.so; do
  tag=$(basename $lib .so)
  IFS=';' read -ra VARS <<< "${QT:-;--d 0}"
  for args in "${VARS[@]}"; do
    echo "## $tag $args" >> gpurun_out/ab.log
    SRNN_LIB=$PWD/$lib timeout 120 python scripts/quick_time.py $args >> gpurun_out/ab.log 2>&1
    if [ -n "$TLINE" ]; then SRNN_LIB=$PWD/$lib timeout 120 python scripts/timeline.py $args >> gpurun_out/ab.log 2>&1; fi
  done
done
done
