#!/bin/bash
# dev tool (run under gpurun): round-2 measurements and ncu evidence for profiles/.
#   1. launch list of the bench command (gpu__time_duration per launch, cold, serialised)
#   2. --set full captures of the level-1 launch of the top kernels (compress + full retrieval of
#      tools/compress_once.py: per-level kernels launch once per level, level 1 last)
#   3. dram traffic of every k_match / k_od_walk launch of one compress (roofline "traffic")
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/compress_once.py 2 full > /dev/null 2>&1 || exit 1
for spec in "k_match 6" "k_od_walk 6" "k_od_sync 6" "k_od_place 6" "k_prevlinks 6" "k_plan 6" "k_emit_syms 6" \
            "k_sim 6" "k_loss_lines 5" "k_bitplanes 6" "k_rows 2" "k_rows 5" "k_decode_cands 0" "k_resolve_all 0" \
            "k_emit 7" "k_merge 6" "k_asm_gather 0"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:^$1\$ --launch-skip $2 -c 1 \
      -o gpurun_out/r2_$1_$2 python tools/compress_once.py 2 full > gpurun_out/r2_$1_$2.log 2>&1
  python tools/ncu_summary.py gpurun_out/r2_$1_$2.ncu-rep > gpurun_out/r2_$1_$2.summary.txt 2>&1
  python tools/ncu_mix.py gpurun_out/r2_$1_$2.ncu-rep 14 >> gpurun_out/r2_$1_$2.summary.txt 2>&1
  case "$1" in k_match|k_od_walk|k_resolve_all|k_loss_lines) ;; *) rm -f gpurun_out/r2_$1_$2.ncu-rep ;; esac
done
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"^(k_match|k_od_walk)$" --csv --log-file gpurun_out/r2_match_traffic.csv \
    python tools/compress_once.py 2 compress > /dev/null 2>&1
du -sh gpurun_out; ls -la gpurun_out | tail -60
