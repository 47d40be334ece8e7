#!/bin/bash
# Build libbte.so of a git revision into abbuild/libbte_<name>.so for same-box A/B
# runs (bench.py with BTE_LIB=abbuild/libbte_<name>.so).  Usage: build_ab.sh REV NAME
set -e
cd "$(dirname "$0")/.."
rev=${1:?rev}; name=${2:?name}
tmp=$(mktemp -d)
git archive "$rev" paper_2305_19400_b200/csrc include | tar -x -C "$tmp"
mkdir -p abbuild
nccl_inc=$(python -c 'import nvidia.nccl,os;print(os.path.join(list(nvidia.nccl.__path__)[0],"include"))' 2>/dev/null || echo /usr/include)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden -I "$tmp/include" -I "$nccl_inc" --expt-relaxed-constexpr \
  -o "abbuild/libbte_$name.so" "$tmp"/paper_2305_19400_b200/csrc/*.cu "$tmp"/paper_2305_19400_b200/csrc/*.cpp -ldl
rm -rf "$tmp"
echo "abbuild/libbte_$name.so"
