#!/bin/bash
# Rebuild all libraries; exit non-zero (and print the nvcc errors) on any failure.
cd "$(dirname "$0")/.." && python -m paper_2009_01614_b200.build > /tmp/rebuild.log 2>&1
rc=$?
if [ $rc -ne 0 ]; then grep -iE " error|error:" -A3 paper_2009_01614_b200/build_isax.log datagen/build_isaxgen.log 2>/dev/null | head -30; echo "BUILD FAILED"; exit 1; fi
grep -h "spill stores" paper_2009_01614_b200/build_isax.log | grep -v " 0 bytes spill" | head -3
echo "build ok"
