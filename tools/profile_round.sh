#!/bin/bash
# dev tool (run under gpurun): the round's measurements and ncu evidence for profiles/.
#   1. bench.py (ours, with the CPU baseline) and bench.py --impl reference
#   2. launch list of the bench command (gpu__time_duration per launch, cold, serialised)
#   3. --set full captures of the level-1 launch of the top kernels (compress + full retrieve)
#   4. dram traffic of every k_match launch of one compress (roofline "traffic")
set -x
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 > gpurun_out/prof_bench.json 2> gpurun_out/prof_bench.err || exit 1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/prof_bench_reference.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python tools/compress_once.py 2 full > /dev/null 2>&1 || exit 1
# compress_once full = warm compress + compress... (see the script); per-level kernels launch once per
# level, level 1 last (index 6); k_rows: 3 quant launches (compress) then 3 recon launches
for spec in "k_match 6" "k_loss_fused 5" "k_prevlinks 6" "k_emit_syms 6" "k_plan 6" "k_bitplanes 6" \
            "k_rows 2" "k_rows 5" "k_decode_cands 0" "k_emit 0" "k_merge 6"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:^$1 --launch-skip $2 -c 1 \
      -o gpurun_out/prof_$1_$2 python tools/compress_once.py 2 full > gpurun_out/prof_$1_$2.log 2>&1
done
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:^k_match \
    -c 7 --csv --log-file gpurun_out/prof_match_traffic.csv python tools/compress_once.py 2 compress > /dev/null 2>&1
ls -la gpurun_out | tail -30
