#!/bin/bash
# A/B timing of library variants on one box: abvar/libsrnn_<tag>.so
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out; rm -f gpurun_out/ab.log
for lib in abvar/libsrnn_*.so; do
  tag=$(basename $lib .so)
  IFS=';' read -ra VARS <<< "${QT:---L 32;--L 32 --bt 4}"
  for args in "${VARS[@]}"; do
    echo "## $tag $args" >> gpurun_out/ab.log
    SRNN_LIB=$PWD/$lib timeout 120 python scripts/quick_time.py $args >> gpurun_out/ab.log 2>&1
    SRNN_LIB=$PWD/$lib timeout 120 python scripts/timeline.py $args >> gpurun_out/ab.log 2>&1
  done
done
