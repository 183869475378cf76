#!/bin/bash
# usage: scripts/sass_probe.sh BAL [K]  -> per-chain-tick SASS mix of the solo kernel's steady stage loop
cd "$(dirname "$0")/.."
V=${1:-2}; K=${2:-1}
nvcc -cubin -o /tmp/sass_probe_$V.cubin scripts/sass_probe.cu -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
  --expt-relaxed-constexpr -I include -DPROBE_V=$V -DPROBE_K=$K -Xptxas -v 2>&1 | grep -E "registers|error" | head -3
python scripts/solo_sass.py /tmp/sass_probe_$V.cubin $K $V | head -2
