mkdir -p gpurun_out/r03j
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for s in "4 32 8 1024 8192" "8 16 8 512 4096" "16 8 8 2048 2048" "8 32 16 1024 4096"; do
  timeout -k 10 600 python scripts/ab_custom.py $s 3 nodyn -DBIFATTN_NO_DYN >> gpurun_out/r03j/ab.jsonl 2>> gpurun_out/r03j/ab.err
done
cat gpurun_out/r03j/ab.jsonl; tail -3 gpurun_out/r03j/ab.err
