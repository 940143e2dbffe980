set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout -k 10 600 python scripts/role_cycles_rows.py mqa gqa > gpurun_out/role_rows.jsonl 2> gpurun_out/role_rows.err
M=sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,smsp__inst_executed_pipe_xu.sum,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,dram__bytes_read.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active
timeout -k 10 300 ncu --metrics $M --clock-control none -k regex:ctx_rows --launch-skip 6 --launch-count 1 --csv python bench.py --config mqa --steps 3 --warmup 3 --no-e2e --no-replicated --no-cpu-baseline --no-stream-peak --no-others --soak 0 > gpurun_out/ncu_rows_mqa.csv 2>&1
