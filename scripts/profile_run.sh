#!/usr/bin/env bash
# ncu evidence for one config (run under gpurun, 1 GPU):
#   bash scripts/profile_run.sh <config> [tag]
# writes gpurun_out/<tag>_launches.csv (every launch, device time),
#        gpurun_out/<tag>_full.ncu-rep (one band-kernel launch, --set full),
#        gpurun_out/<tag>_pipes.csv   (pipe utilisation, shared-atomic
#        wavefronts/conflicts, occupancy, DRAM bytes of the band kernel AND of
#        the L2-flush kernel that follows it: the flush evicts the band
#        kernel's dirty lines, so band write traffic = band + flush - 256 MiB)
set -u
cfg=$1; tag=${2:-$1}
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config $cfg"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}_launches.csv $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"band_(sorted_)?kernel" -s 3 -c 1 \
  -o gpurun_out/${tag}_full -f $B > /dev/null 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active
M=$M,sm__inst_executed.sum,sm__inst_executed.avg.per_cycle_active
M=$M,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active
M=$M,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active
M=$M,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.sum
M=$M,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum
M=$M,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed
timeout 900 ncu --metrics $M --clock-control none -c 16 --csv --log-file gpurun_out/${tag}_pipes.csv $B > /dev/null 2>&1
ls -la gpurun_out/${tag}_*
