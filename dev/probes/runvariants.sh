#!/bin/bash
# on the GPU box: run a command once per dev/variants/libsgiga_*.so (copied
# over the in-tree library), e.g. runvariants.sh 'python dev/probes/asm_once.py cfg5'
cd "$(dirname "$0")/../.."
cp paper_1707_09598_b200/libsgiga.so /tmp/libsgiga_orig.so
for v in dev/variants/libsgiga_*.so; do
  cp "$v" paper_1707_09598_b200/libsgiga.so
  echo "== $(basename $v)"
  eval "$1"
done
cp /tmp/libsgiga_orig.so paper_1707_09598_b200/libsgiga.so
