#!/bin/bash
# Build locally (must succeed), then run the given command on the GPU box.
cd /root/repo || exit 1
python paper_2110_14007_b200/build.py > /tmp/build.log 2>&1 || { echo "BUILD FAILED"; grep -m5 error /tmp/build.log; exit 1; }
exec timeout 3000 /usr/local/graft/bin/gpurun --timeout "${GPU_TIMEOUT:-1200}" -- "$@"
