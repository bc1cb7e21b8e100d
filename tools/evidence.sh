#!/bin/bash
# Round evidence: bench line, ncu launch list, and one --set full capture each of the
# worker step (round 0 = seeding, round 1 = steady) and of f(C,X). Run under gpurun.
cd $GRAFT_REPO_ROOT
P=${1:-r1}
python bench.py > gpurun_out/${P}_bench.log 2>&1 || { tail -20 gpurun_out/${P}_bench.log; exit 1; }
tail -1 gpurun_out/${P}_bench.log > gpurun_out/${P}_bench.json
python bench.py --impl reference > gpurun_out/${P}_bench_ref.log 2>&1; tail -1 gpurun_out/${P}_bench_ref.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${P}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-configs > gpurun_out/${P}_ncu_launches.log 2>&1
for spec in "worker_step:0:step_round0" "worker_step:1:step_round1" "objective:0:objective"; do
  IFS=: read kre skip name <<< "$spec"
  ncu --set full --import-source on --clock-control none -k regex:$kre -s $skip -c 1 -f -o gpurun_out/${P}_$name \
      python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e --no-configs > gpurun_out/${P}_${name}_ncu.log 2>&1
done
ls -la gpurun_out/ | grep $P
