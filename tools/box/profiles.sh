#!/bin/bash
# Refresh the profiles/ evidence for a tag: bench lines (config 1 default, 0, 3),
# the serialised ncu launch list of one config-1 registration, and an
# ncu --set full capture of the full-resolution loop kernels.
TAG=$1
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
python bench.py --config 0 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_config0.json 2>/dev/null; echo "c0 rc=$?"
python bench.py --config 3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_config3.json 2>/dev/null; echo "c3 rc=$?"
python tools/prof_one.py 1 f32 1 > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/${TAG}_launches.csv python tools/prof_one.py 1 f32 0 > gpurun_out/${TAG}_ncu_launches.log 2>&1; echo "launches rc=$?"
python tools/prof_level.py 160 192 224 4 > gpurun_out/${TAG}_pl.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_zm2" -s 10 -c 5 \
    -o gpurun_out/${TAG}_full_f32 python tools/prof_level.py 160 192 224 4 > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "full rc=$?"
