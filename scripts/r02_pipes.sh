set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
M=sm__inst_executed_pipe_xu.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fmaheavy.sum,sm__inst_executed_pipe_lsu.sum,sm__inst_executed_pipe_tmem.sum,sm__inst_executed_pipe_uniform.sum,smsp__inst_executed.sum,sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active
for c in mha7b_b32 mha7b_b32_fp8; do
timeout -k 10 300 ncu --metrics $M --clock-control none -k regex:bif_tc --launch-skip 6 --launch-count 1 --csv python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-replicated --no-cpu-baseline --no-stream-peak --no-others --soak 0 > gpurun_out/pipes_$c.csv 2>&1
done
