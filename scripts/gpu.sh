#!/bin/bash
# Build in-tree (the .so travels with the snapshot), then run a command on a B200.
# usage: scripts/gpu.sh TIMEOUT 'command'
set -e
cd /root/repo
python paper_2501_15348_b200/build.py | grep -E "error|failed|linked" || true
exec /usr/local/graft/bin/gpurun --timeout "$1" -- "$2"
