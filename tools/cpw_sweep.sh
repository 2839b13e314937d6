#!/bin/bash
# dev tool (run under gpurun): rebuild inflate.cu with -DIPCG_CPW=c for each c and profile
for c in "$@"; do
  touch paper_2502_04093_b200/csrc/inflate.cu
  python -c "import sys; sys.path.insert(0,'.'); from paper_2502_04093_b200 import build as b; b.PER_FILE['inflate.cu']=['-D'+'$c']; b.build()" || exit 1
  echo "$c"; python tools/planeprof.py 2 1 - inflate 2>&1 | grep "inflate " | cut -c1-120
done
