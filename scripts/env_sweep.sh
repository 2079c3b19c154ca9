#!/bin/bash
# Timing under environment knobs: ENVS="A=1 B=2;A=3" (one quick_time per setting and QT arg set)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out; OUT=gpurun_out/${TAG:-envs}.log; rm -f $OUT
IFS=';' read -ra ES <<< "${ENVS:-X=0}"
IFS=';' read -ra VARS <<< "${QT:-}"
[ ${#VARS[@]} -eq 0 ] && VARS=("")
for r in $(seq ${ROUNDS:-1}); do
for e in "${ES[@]}"; do
  for args in "${VARS[@]}"; do
    echo "## $e $args" >> $OUT
    env $e ${LIBENV} timeout 120 python scripts/quick_time.py $args >> $OUT 2>&1
  done
done
done
