mkdir -p gpurun_out/r03v
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in mqa gqa long; do timeout -k 10 600 python scripts/kernel_shares.py $c "" paper_2403_08845_b200/libbifattn_rows1.so >> gpurun_out/r03v/shares.jsonl 2>>gpurun_out/r03v/err.txt; done
cat gpurun_out/r03v/shares.jsonl; tail -3 gpurun_out/r03v/err.txt
