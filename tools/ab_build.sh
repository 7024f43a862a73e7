#!/bin/bash
# A/B variants of libhgm.so: tools/ab_build.sh name "-DX=0 -DY=1" ...  (pairs)
while [ $# -ge 2 ]; do
  HGM_BUILD_TAG=$1 HGM_BUILD_DEFS="$2" python -c "from paper_1505_00581_b200 import build as B; print(B.build())" || exit 1
  shift 2
done
