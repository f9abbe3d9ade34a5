#!/bin/bash
# Build (fail loudly) then run a command on the B200 box via gpurun.
# usage: tools/gpu.sh <timeout-seconds> '<command>'
set -e
cd /root/repo
python paper_1305_1070_b200/build.py > /tmp/build.log 2>&1 || { grep -E "error" /tmp/build.log | head -20; echo "BUILD FAILED"; exit 1; }
timeout $(( $1 + 1500 )) /usr/local/graft/bin/gpurun --timeout "$1" -- "$2"
