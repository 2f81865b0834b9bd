#!/bin/bash
# build libcakf.so from the repo root; non-zero exit (and the compiler output) on any error
cd "$(dirname "$0")/.." || exit 1
out=$(python -m paper_2405_08971_b200.build 2>&1); rc=$?
if [ $rc -ne 0 ] || echo "$out" | grep -qE "error|Error"; then echo "$out" | grep -E "error|Error" | head -20; exit 1; fi
echo "build ok"
