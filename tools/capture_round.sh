#!/bin/bash
# One-GPU capture of the round's evidence into gpurun_out/$1 (run under gpurun):
#   full ncu capture of the two streaming kernels at T=1e8 -> summary + per-launch DRAM traffic (which
#   bench.py then reads from profiles/ncu_traffic.json), the bench line, the ncu launch list of the same
#   bench command, full ncu captures of the config 3 (D=64) and config 4 (B=1024, D=16) kernels with
#   tensor-pipe / FMA-pipe activity, per-config device times, phase stamps and split-phase per-rank timing.
set -x
OUT=gpurun_out/$1; mkdir -p $OUT
ncu -f --set full --import-source on --clock-control none -k regex:hmm_stream_kernel -c 2 -o /tmp/stream_full python tools/run_once.py 1e8 > $OUT/ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/stream_full.ncu-rep $OUT/ncu_traffic.json 1e8 > $OUT/ncu_full_summary.json 2>&1
cp $OUT/ncu_traffic.json profiles/ncu_traffic.json
python bench.py > $OUT/bench.json 2> $OUT/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-configs > $OUT/launches.log 2>&1
ncu -f --set full --clock-control none -c 12 -o /tmp/config3_full python tools/run_config3.py > $OUT/config3_ncu.log 2>&1
python tools/ncu_summary.py /tmp/config3_full.ncu-rep > $OUT/config3_ncu_summary.json 2>&1
ncu -f --set full --clock-control none -c 4 -o /tmp/config4_full python tools/run_config4.py > $OUT/config4_ncu.log 2>&1
python tools/ncu_summary.py /tmp/config4_full.ncu-rep > $OUT/config4_ncu_summary.json 2>&1
python tools/time_configs.py big > $OUT/configs.txt 2>&1
python tools/stream_phases.py > $OUT/phases.txt 2>&1
python tools/phase_timers.py 1000000 > $OUT/phases_T1e6.txt 2>&1
python tools/dist_rank_timing.py > $OUT/dist_rank_timing.txt 2>&1
python tools/batchseq_crossover.py > $OUT/batchseq_crossover.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $OUT/config3_launches.csv python tools/run_config3.py > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $OUT/config4_launches.csv python tools/run_config4.py > /dev/null 2>&1
