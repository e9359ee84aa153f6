#!/bin/bash
# build libsgiga.so; non-zero exit (and the nvcc error) on failure
python -c "from paper_1707_09598_b200 import build as B; B.build(verbose=True)" > /tmp/build.log 2>&1
rc=$?
if [ $rc -ne 0 ]; then grep -B2 -A6 "error" /tmp/build.log | head -30; exit 1; fi
grep -A3 "_ZN5sgiga15k_assemble_fastILi3ELi[45]" paper_1707_09598_b200/_build/k_assembly_fast.ptxas.log | grep -i "registers\|spill"
