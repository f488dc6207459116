#!/bin/bash
# tools/g.sh '<command>' [timeout]  -- run a command on the GPU box from the repo root
cd /root/repo || exit 1
T=${2:-1200}
timeout $((T + 600)) /usr/local/graft/bin/gpurun --timeout $T -- "$1" > gpurun_out/last_call.txt 2>&1
tail -1 gpurun_out/last_call.txt
