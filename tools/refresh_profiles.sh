#!/bin/bash
# Copies the outputs of tools/collect_profiles.sh from gpurun_out/ into profiles/ and
# derives the text summaries (runs here, without a GPU). usage: tools/refresh_profiles.sh r1
TAG=${1:-r1}
for f in bench_stage.json bench_split.json bench_fused.json bench_stage_f32.json bench_reference.json \
         bench_baroclinic.json bench_baroclinic_4e8.json launches.csv launches_split.csv smi.csv \
         ubench_fp64_ubench.txt ubench_fp64_operands_ubench.txt ubench_smem_ubench.txt \
         order_precision_sweep.jsonl error_survey.txt; do
  cp gpurun_out/${TAG}_$f profiles/${TAG}_$f
done
python tools/ncu_summary.py gpurun_out/${TAG}_full_stage.ncu-rep gpurun_out/${TAG}_full_split.ncu-rep > profiles/${TAG}_ncu_full_summary.txt 2>&1
python tools/ncu_phases.py gpurun_out/${TAG}_full_stage.ncu-rep > profiles/${TAG}_ncu_stage_phases.txt 2>&1
python - <<PY
import csv
rows = list(csv.reader(open('gpurun_out/${TAG}_full_split_source.csv')))
out, keep, n = [], False, 0
for r in rows:
    if r and r[0] == 'Kernel Name':
        n += 1
        keep = n == 1
    if keep:
        out.append(r)
csv.writer(open('/tmp/k1_source.csv', 'w')).writerows(out)
PY
(echo "stage kernel:"; python tools/ncu_fp64_cycles.py gpurun_out/${TAG}_full_stage_source.csv; python tools/ncu_stalls.py gpurun_out/${TAG}_full_stage_source.csv
 echo; echo "split path, volume kernel:"; python tools/ncu_fp64_cycles.py /tmp/k1_source.csv; python tools/ncu_stalls.py /tmp/k1_source.csv) > profiles/${TAG}_ncu_stage_pipe_cycles.txt
# profiles/traffic.json comes from tools/collect_traffic.py (one ncu pass per sweep point)
