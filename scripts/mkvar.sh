#!/bin/bash
# Build A/B variants of libsrnn.so: VARS="tag1=-DX -DY;tag2=-DZ" -> abvar/libsrnn_<tag>.so
# (then restores the plain build).  Used with scripts/ab.sh on the GPU box.
cd "$(dirname "$0")/.."
mkdir -p abvar
IFS=';' read -ra VS <<< "$VARS"
for v in "${VS[@]}"; do
  tag=${v%%=*}; fl=${v#*=}
  SRNN_NVCC_FLAGS="$fl" python -c "from paper_1804_10223_b200 import build as b; b.build()" || exit 1
  cp paper_1804_10223_b200/libsrnn.so abvar/libsrnn_${tag}.so
  echo "built $tag ($fl)"
done
python -c "from paper_1804_10223_b200 import build as b; b.build()"
