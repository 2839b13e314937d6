#!/bin/bash
# dev tool (run under gpurun): where a small field's compress / retrieval time goes --
# host phase marks (IPCG_DEBUG_TIMING), device timeline marks (IPCG_DEBUG_TIMELINE) and the
# per-kernel launch list of one cfg1 compress + full retrieval.
O=gpurun_out/small; mkdir -p $O
IPCG_DEBUG_TIMING=1 python tools/small_calls.py 1 > $O/timing1.txt 2>&1
IPCG_DEBUG_TIMING=1 python tools/small_calls.py 3 > $O/timing3.txt 2>&1
IPCG_DEBUG_TIMELINE=1 python tools/small_calls.py 1 > $O/timeline1.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches1.csv \
    python tools/compress_once.py 1 full > /dev/null 2>&1
python tools/launch_summary.py $O/launches1.csv > $O/launches1_summary.txt
