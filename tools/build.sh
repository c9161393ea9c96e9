#!/bin/bash
# build libchg.so from anywhere; prints compiler errors and a one-line verdict
cd "$(dirname "$0")/.." || exit 1
out=$(python paper_2412_20796_b200/build.py 2>&1)
rc=$?
echo "$out" | grep -E " error|error:" -A3 | head -30
if [ $rc -eq 0 ] && ! echo "$out" | grep -q " error"; then echo "BUILD OK"; else echo "BUILD FAILED (rc=$rc)"; echo "$out" | tail -5; fi
