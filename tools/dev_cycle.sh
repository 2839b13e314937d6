#!/bin/bash
# dev tool: build here (abort on error), then GPU parity + probe in one gpurun call.
# usage: tools/dev_cycle.sh TAG [extra remote command]
set -e
cd /root/repo
tag=$1; shift || true
python -c "import sys; sys.path.insert(0,'.'); from paper_2502_04093_b200 import build as b; b.build(verbose=False)" 2>&1 | grep -E "error" && { echo BUILD FAILED; exit 1; }
extra="$*"
timeout 2400 /usr/local/graft/bin/gpurun --timeout 1200 -- "mkdir -p gpurun_out; python -m pytest tests -m gpu -x -q > gpurun_out/parity_$tag.log 2>&1; tail -2 gpurun_out/parity_$tag.log; python tools/probe.py 2 > gpurun_out/probe_$tag.log 2>&1; grep -A1 'compress wall' gpurun_out/probe_$tag.log | tail -2; grep -A1 'retrieve rel 0.0001' gpurun_out/probe_$tag.log; $extra" 2>&1 | grep -v "^\[gpurun\] sending"
