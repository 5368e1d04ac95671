#!/bin/bash
# Build libtvreg from the working tree with one source file replaced and / or extra nvcc flags
# (A/B timing with TVR_LIB_PATH).  usage: scripts/build_variant.sh <out.so> [<file.cu> <replacement>] [-- nvcc flags]
set -e
OUT=$(realpath -m $1); shift
D=$(mktemp -d)
mkdir -p $D/a/b
cp -r paper_1105_4002_b200/csrc $D/a/b/
cp -r include $D/a/include
if [ "$1" != "" ] && [ "$1" != "--" ]; then cp $2 $D/a/b/csrc/$1; shift 2; fi
[ "$1" == "--" ] && shift
INC=$(python -c "import sys; sys.path.insert(0,'$PWD'); from paper_1105_4002_b200 import _build; print(_build.nccl_dirs()[0])")
LIBD=$(python -c "import sys; sys.path.insert(0,'$PWD'); from paper_1105_4002_b200 import _build; print(_build.nccl_dirs()[1])")
cd $D/a/b
for f in csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 "$@" -Xcompiler -fPIC -I $INC -c $f -o $f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT csrc/*.o -L $LIBD -l:libnccl.so.2 -Xlinker -rpath=$LIBD
rm -rf $D
echo $OUT
