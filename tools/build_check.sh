#!/bin/bash
# rebuild the CUDA library from the repo root; fail loudly
cd "$(dirname "$0")/.." || exit 1
python -m paper_2105_01827_b200.build --force > /tmp/gala_build.log 2>&1 || { grep -E "error" -A3 /tmp/gala_build.log | head -40; exit 1; }
echo "build ok"
