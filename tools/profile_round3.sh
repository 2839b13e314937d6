#!/bin/bash
# dev tool (run under gpurun): the round-2 (final session) measurements and ncu evidence for profiles/.
#   1. bench.py (ours, CPU baseline included) and bench.py --impl reference
#   2. per-config table (all five BASELINE configs)
#   3. launch list of the bench command (gpu__time_duration per launch, cold, serialised)
#   4. --set full captures of the level-1 launch of the top kernels (tools/compress_once.py 2 full:
#      per-level kernels launch once per level, level 1 last) and of the retrieval kernels
#   5. dram traffic of every k_match / k_od_walk launch of one compress (roofline "traffic")
set -x
mkdir -p gpurun_out/p3
O=gpurun_out/p3
python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; tail -2 $O/gputests.log
python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err || exit 1
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
python tools/config_table.py > $O/configs.jsonl 2> $O/configs.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python tools/launch_summary.py $O/launches.csv > $O/launches_summary.txt
for spec in "k_match 6" "k_prevlinks_pair 6" "k_plan 6" "k_od_walk 2" "k_emit_syms 6" "k_sim 6" "k_loss_lines 5" \
            "k_bitplanes 6" "k_rows 2" "k_rows 5" "k_decode_cands 0" "k_resolve_all 0" "k_validate 0" "k_merge 6"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:^$1\$ --launch-skip $2 -c 1 \
      -o $O/$1_$2 python tools/compress_once.py 2 full > $O/$1_$2.log 2>&1
  python tools/ncu_summary.py $O/$1_$2.ncu-rep > $O/$1_$2.summary.txt 2>&1
  python tools/ncu_mix.py $O/$1_$2.ncu-rep 14 >> $O/$1_$2.summary.txt 2>&1
  case "$1" in k_match|k_resolve_all|k_decode_cands|k_plan) ;; *) rm -f $O/$1_$2.ncu-rep ;; esac
done
# inflate's k_emit (deflate has a kernel of the same name: select by the mangled file scope)
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:inflate_cu.*k_emit \
    -c 1 -o $O/inflate_k_emit python tools/compress_once.py 2 full > $O/inflate_k_emit.log 2>&1
python tools/ncu_summary.py $O/inflate_k_emit.ncu-rep > $O/inflate_k_emit.summary.txt 2>&1
rm -f $O/inflate_k_emit.ncu-rep
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"^(k_match|k_od_walk)$" --csv --log-file $O/match_traffic.csv \
    python tools/compress_once.py 2 compress > /dev/null 2>&1
du -sh $O; ls -la $O | tail -60
