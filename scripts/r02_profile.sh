# round-2 profile: timeline of the fused kernel, default bench line, ncu full set of the C2b kernel
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 600 python scripts/timeline.py mha7b_b32 mha7b_b32_fp8 mha7b_b16 > gpurun_out/timeline.jsonl 2> gpurun_out/timeline.err
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bif_tc_kernel --launch-skip 8 --launch-count 1 -o gpurun_out/prof_b32 \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-replicated --no-cpu-baseline --no-stream-peak --no-others --soak 0 > gpurun_out/ncu_b32.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bif_tc_kernel --launch-skip 8 --launch-count 1 -o gpurun_out/prof_fp8 \
  python bench.py --config mha7b_b32_fp8 --steps 3 --warmup 3 --no-e2e --no-replicated --no-cpu-baseline --no-stream-peak --no-others --soak 0 > gpurun_out/ncu_fp8.log 2>&1
