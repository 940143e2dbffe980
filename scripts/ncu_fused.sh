mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
B="python bench.py --steps 3 --warmup 3 --soak 0 --no-e2e --no-replicated --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bif_tc_kernel -s 3 -c 1 -o gpurun_out/prof_fused2 $B > gpurun_out/ncu_fused2.log 2>&1
tail -3 gpurun_out/ncu_fused2.log
