#!/bin/bash
# Rebuild libgcm.so in-tree; exit non-zero (and show the errors) if it fails.
cd "$(dirname "$0")/.." || exit 1
out=$(python paper_1011_1173_b200/_build.py 2>&1) || { echo "$out" | grep -E "error" | head -20; echo "BUILD FAILED"; exit 1; }
echo "built $(ls -la --time-style=+%T paper_1011_1173_b200/lib/libgcm.so | awk '{print $6}')"
