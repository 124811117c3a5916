#!/usr/bin/env bash
set -u
TAG=${1:-r2p}
OUT=gpurun_out
ARGS1="--config c5 --images 512 --templates 64 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 120 python bench.py $ARGS1 > $OUT/plain_${TAG}.json 2>&1 && \
timeout 300 ncu --metrics smsp__inst_executed.sum,sm__cycles_elapsed.avg,smsp__cycles_active.avg,smsp__inst_executed_pipe_lsu.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
   --clock-control none -k regex:"k_step" -c 4 --csv --log-file $OUT/ncu_m_${TAG}.csv python bench.py $ARGS1 > $OUT/ncu_m_${TAG}.log 2>&1
echo "ncu rc $?"
grep -E "ERROR" $OUT/ncu_m_${TAG}.log | head -3
FTK_S23=0 timeout 300 ncu --metrics smsp__inst_executed.sum,sm__cycles_elapsed.avg,smsp__cycles_active.avg,smsp__inst_executed_pipe_lsu.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed \
   --clock-control none -k regex:"k_step" -c 6 --csv --log-file $OUT/ncu_m_sep_${TAG}.csv python bench.py $ARGS1 > $OUT/ncu_m_sep_${TAG}.log 2>&1
echo "ncu sep rc $?"
echo done
