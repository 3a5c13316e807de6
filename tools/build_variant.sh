#!/bin/bash
# Build the library with one csrc file replaced (A/B experiments):
#   tools/build_variant.sh <replacement.cu> <target file name in csrc> <out.so>
set -e
REPO=$(cd "$(dirname "$0")/.." && pwd)
T=$(mktemp -d)
cp "$REPO"/paper_1802_06263_b200/csrc/* "$T"/
cp "$1" "$T/$2"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
  -I "$REPO/include" -I "$T" $EXTRA -o "$3" "$T"/*.cu -lcudart
rm -rf "$T"
