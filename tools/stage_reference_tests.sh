#!/bin/bash
# Copy the reference package's own test suite into the git-ignored
# baseline/_ref/tests so it ships to the GPU box with the gpurun snapshot
# (tests/reference_suite/run_reference_suite.py runs it against this package).
set -eu
repo=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$repo/baseline/_ref"
rm -rf "$repo/baseline/_ref/tests"
cp -r /root/reference/pkg/tests "$repo/baseline/_ref/tests"
echo "staged $(ls "$repo/baseline/_ref/tests" | wc -l) files into baseline/_ref/tests"
