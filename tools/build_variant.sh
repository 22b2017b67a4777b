#!/bin/bash
# build a variant of libidconv.so with extra -D flags into tools/var_<name>.so (experiments only)
set -e
name=$1; shift
cd "$(dirname "$0")/.."
NCCL=$(python -c "import nvidia.nccl,os;print(list(nvidia.nccl.__path__)[0])")
mkdir -p /tmp/var_$name
for f in paper_1008_1366_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -Iinclude -I$NCCL/include "$@" -c $f -o /tmp/var_$name/$b.o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/var_$name.so /tmp/var_$name/*.o -lcudart -L$NCCL/lib -l:libnccl.so.2 -Xlinker -rpath=$NCCL/lib
echo built tools/var_$name.so
