#!/bin/bash
# Build libtvreg from a git revision into an alternate .so (A/B timing with TVR_LIB_PATH).
# usage: scripts/build_rev.sh <rev> <out.so>
set -e
REV=$1; OUT=$(realpath -m $2)
D=$(mktemp -d)
git archive $REV paper_1105_4002_b200/csrc include | tar -x -C $D
INC=$(python -c "import sys; sys.path.insert(0,'$PWD'); from paper_1105_4002_b200 import _build; print(_build.nccl_dirs()[0])")
LIBD=$(python -c "import sys; sys.path.insert(0,'$PWD'); from paper_1105_4002_b200 import _build; print(_build.nccl_dirs()[1])")
cd $D
for f in paper_1105_4002_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -I include -I $INC -c $f -o $f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT paper_1105_4002_b200/csrc/*.o -L $LIBD -l:libnccl.so.2 -Xlinker -rpath=$LIBD
rm -rf $D
echo $OUT
