# round-2 GPU check: build, GPU tests, bench line, tensor-pipe counters per config
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -rA > gpurun_out/pytest_gpu.txt 2>&1
grep -E "rows: max_abs|plan-covering|b32-n4" gpurun_out/pytest_gpu.txt > gpurun_out/parity_full.txt
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
M=sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tc.sum,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed
for c in mha7b_b32 gqa mqa long; do
  timeout 300 ncu --metrics $M --clock-control none --cache-control all -k regex:"bif_tc|ctx_rows|merge" --launch-skip 6 --launch-count 4 --csv \
    python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-replicated --no-cpu-baseline --soak 0 > gpurun_out/tc_$c.csv 2> gpurun_out/tc_$c.err
done
