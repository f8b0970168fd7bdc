#!/bin/bash
# Build everything locally first (abort on failure), then run the given command on a B200.
# usage: tools/gpu.sh TIMEOUT_S 'command'
set -e
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" > /tmp/gpu_build.log 2>&1 || { tail -20 /tmp/gpu_build.log; echo BUILD FAILED; exit 1; }
mkdir -p gpurun_out
timeout $(( $1 + 600 )) /usr/local/graft/bin/gpurun --timeout "$1" -- "mkdir -p gpurun_out; $2"
