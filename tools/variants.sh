#!/bin/bash
# dev tool: build library variants of one source file under different -D flags into _var/<name>.so
#   tools/variants.sh inflate.cu name1 "-DA=1 -DB=2" name2 "-DA=0" ...
# then on the GPU: cp _var/<name>.so paper_2502_04093_b200/libipcomp_b200.so before each run.
set -e
src=$1; shift
mkdir -p _var
while [ $# -gt 1 ]; do
  name=$1; flags=$2; shift 2
  rm -f paper_2502_04093_b200/_build/$src.o paper_2502_04093_b200/libipcomp_b200.so
  IPCG_NVCC_EXTRA="$flags" python -c "from paper_2502_04093_b200 import build as b; b.build(force=False)"
  cp paper_2502_04093_b200/libipcomp_b200.so _var/$name.so
done
rm -f paper_2502_04093_b200/_build/$src.o paper_2502_04093_b200/libipcomp_b200.so
python -c "from paper_2502_04093_b200 import build as b; b.build()"
