mkdir -p gpurun_out/r03o
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout -k 10 600 python scripts/role_cycles_rows.py mqa gqa long > gpurun_out/r03o/role_cycles_rows.jsonl 2> gpurun_out/r03o/rc.err
cat gpurun_out/r03o/role_cycles_rows.jsonl; tail -3 gpurun_out/r03o/rc.err
