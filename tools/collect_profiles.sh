#!/bin/bash
# Runs on the GPU box (via gpurun): bench lines, ncu launch list and ncu --set
# full captures that profiles/ is built from. Output goes to gpurun_out/.
set -u
OUT=gpurun_out
mkdir -p $OUT
TAG=${1:-r1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw,power.limit --format=csv > $OUT/${TAG}_smi.csv
timeout 400 python bench.py > $OUT/${TAG}_bench_stage.json 2> $OUT/${TAG}_bench_stage.err
timeout 300 python bench.py --path split --no-cpu-baseline > $OUT/${TAG}_bench_split.json 2> $OUT/${TAG}_bench_split.err
timeout 300 python bench.py --path fused --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench_fused.json 2> $OUT/${TAG}_bench_fused.err
timeout 300 python bench.py --precision f32 --no-cpu-baseline > $OUT/${TAG}_bench_stage_f32.json 2> $OUT/${TAG}_bench_f32.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 1 > $OUT/${TAG}_bench_reference.json 2> $OUT/${TAG}_bench_reference.err
timeout 300 python bench.py --case baroclinic --no-cpu-baseline > $OUT/${TAG}_bench_baroclinic.json 2> $OUT/${TAG}_bench_baroclinic.err
timeout 600 python bench.py --case baroclinic --base 12 4 2 --steps 3 --no-cpu-baseline --no-e2e > $OUT/${TAG}_bench_baroclinic_4e8.json 2> $OUT/${TAG}_bench_baroclinic_4e8.err
timeout 900 python tools/sweep_probe.py > $OUT/${TAG}_order_precision_sweep.jsonl 2> $OUT/${TAG}_sweep.err
timeout 900 python tools/error_survey.py > $OUT/${TAG}_error_survey.txt 2>&1
# every launch of the default bench command with its device time
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file $OUT/${TAG}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/${TAG}_ncu_launches.log 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file $OUT/${TAG}_launches_split.csv python bench.py --path split --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/${TAG}_ncu_launches_split.log 2>&1
# full captures at the bench size (configs[1]); one launch each
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rhs_kernel -s 16 -c 1 \
  -o $OUT/${TAG}_full_stage python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/${TAG}_ncu_full_stage.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rhs_kernel|axpy_kernel" -s 45 -c 3 \
  -o $OUT/${TAG}_full_split python bench.py --path split --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/${TAG}_ncu_full_split.log 2>&1
for r in ${TAG}_full_stage ${TAG}_full_split; do
  ncu -i $OUT/$r.ncu-rep --page source --csv > $OUT/${r}_source.csv 2>/dev/null
done
# micro-benchmarks the design notes cite (FP64 pipe, operand count, shared memory)
for u in fp64_ubench fp64_operands_ubench smem_ubench; do
  [ -x tools/ubench/$u ] && timeout 120 ./tools/ubench/$u > $OUT/${TAG}_ubench_$u.txt 2>&1
done
ls -la $OUT | tail -30
