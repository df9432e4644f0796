#!/bin/bash
# One round of measurement evidence on a B200 (run under gpurun from the repo root):
#   tools/evidence.sh r01f
# bench line, all configs, the bench's ncu launch list, one ncu --set full
# capture of the headline step and one of every kernel family.  Every ncu run
# follows a clean (non-ncu) run of the same command.
set -u
P=${1:?round tag}
O=gpurun_out
mkdir -p $O
python bench.py > $O/${P}_bench.json 2> $O/${P}_bench.err; echo "bench rc=$?"
python tools/bench_configs.py --out $O/${P}_configs.json > $O/${P}_configs.log 2>&1; echo "configs rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${P}_launches_raw.csv \
    python bench.py --steps 2 --warmup 3 > $O/${P}_ncu_bench.log 2>&1; echo "ncu launches rc=$?"
python tools/profile_step.py > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:mumode_tma_kernel -c 3 -f -o $O/${P}_step \
    python tools/profile_step.py > $O/${P}_ncu_step.log 2>&1; echo "ncu step rc=$?"
python tools/profile_kernels.py > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -f -o $O/${P}_kernels \
    python tools/profile_kernels.py > $O/${P}_ncu_kernels.log 2>&1; echo "ncu kernels rc=$?"
# summaries (the .ncu-rep files are too large to bring back)
python tools/ncu_summary.py $O/${P}_step.ncu-rep $O/${P}_launches_raw.csv $O/${P} > $O/${P}_summary.log 2>&1
python tools/kernel_evidence.py $O/${P}_kernels.ncu-rep $O/${P}_kernels >> $O/${P}_summary.log 2>&1
ncu -i $O/${P}_step.ncu-rep --page source --csv 2>/dev/null | gzip > $O/${P}_step_source.csv.gz
ncu -i $O/${P}_step.ncu-rep --page details --csv 2>/dev/null | gzip > $O/${P}_step_details.csv.gz
mkdir -p /tmp/ncu_reps && mv $O/*.ncu-rep /tmp/ncu_reps/ 2>/dev/null
echo "summaries done"; du -sh $O
