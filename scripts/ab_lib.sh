#!/bin/bash
# Build the library of git revision $1 into ab/libedl_$1.so (for EDL_LIB=... A/B
# runs on one box against the working tree's build). Run from the repo root.
set -e
rev=${1:?revision}
tmp=$(mktemp -d)
git archive "$rev" paper_2207_06667_b200/csrc include | tar -x -C "$tmp"
mkdir -p ab
objs=()
for f in "$tmp"/paper_2207_06667_b200/csrc/*.cu; do
  o="$tmp/$(basename "$f" .cu).o"
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
    --expt-relaxed-constexpr -I"$tmp/include" -c "$f" -o "$o" &
  objs+=("$o")
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "ab/libedl_$rev.so" "${objs[@]}" -lrt
rm -rf "$tmp"
echo "ab/libedl_$rev.so"
