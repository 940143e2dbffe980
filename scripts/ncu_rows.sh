mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
B="python bench.py --steps 3 --warmup 3 --soak 0 --no-e2e --no-replicated --no-cpu-baseline"
BIFATTN_CTX_ROWS=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:ctx_rows -s 3 -c 1 -o gpurun_out/prof_r01b_rows_gqa $B --config gqa > gpurun_out/ncu_rows_gqa.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ctx_rows -s 3 -c 1 -o gpurun_out/prof_r01b_rows_mqa $B --config mqa > gpurun_out/ncu_rows_mqa.log 2>&1
tail -2 gpurun_out/ncu_rows_gqa.log gpurun_out/ncu_rows_mqa.log
