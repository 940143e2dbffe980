# round-3 evidence: default bench line, GPU tests, smoke, ncu launch list of the
# bench command, ncu full-set captures of the dominant kernels (exported to CSV pages on the
# box: the reports themselves exceed gpurun's copy-back limit), timelines
set -x
mkdir -p gpurun_out/r03final3
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r03final3/build.txt 2>&1
timeout -k 10 900 python bench.py > gpurun_out/r03final3/bench.json 2> gpurun_out/r03final3/bench.err
timeout -k 10 900 python -m pytest tests -m gpu -q -x --timeout 120 -rA > gpurun_out/r03final3/pytest_gpu.txt 2>&1
grep -E "rows: max_abs|plan-covering|b32-n4|mha7b_b32_fp8: all" gpurun_out/r03final3/pytest_gpu.txt > gpurun_out/r03final3/parity_full.txt
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r03final3/smoke.txt 2>&1
# (compute-sanitizer is closed on this pool in round 3: runs under it are refused)
timeout -k 10 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
  python bench.py --steps 5 --warmup 3 --no-e2e --no-replicated --no-cpu-baseline --no-stream-peak --no-others --soak 0 > gpurun_out/r03final3/launches.csv 2>&1
for c in mha7b_b32:bif_tc:b32 mha7b_b32_fp8:bif_tc:fp8 mqa:ctx_rows_kernel:mqa gqa:ctx_rows_kernel:gqa long:bif_tc:long long:ctx_rows2:long_rows2; do
  cfg=${c%%:*}; rest=${c#*:}; k=${rest%%:*}; tag=${rest#*:}
  timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 6 --launch-count 1 -o /tmp/prof_$tag \
    python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-replicated --no-cpu-baseline --no-stream-peak --no-others --soak 0 > gpurun_out/r03final3/ncu_$tag.log 2>&1
  for page in details raw; do ncu -i /tmp/prof_$tag.ncu-rep --page $page --csv > gpurun_out/r03final3/prof_$tag.$page.csv 2>/dev/null; done
  rm -f /tmp/prof_$tag.ncu-rep
done
timeout -k 10 600 python scripts/timeline.py mha7b_b32 mha7b_b16 > gpurun_out/r03final3/timeline.jsonl 2> gpurun_out/r03final3/timeline.err
timeout -k 10 600 python scripts/role_cycles_rows.py mqa gqa > gpurun_out/r03final3/role_cycles_rows.jsonl 2> gpurun_out/r03final3/role_cycles_rows.err
MT_CFG=mha7b_b32 timeout -k 10 300 python scripts/bench_multitoken.py > gpurun_out/r03final3/multitoken.jsonl 2> gpurun_out/r03final3/multitoken.err
du -sh gpurun_out
