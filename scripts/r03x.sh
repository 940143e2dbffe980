mkdir -p gpurun_out/r03x
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout -k 10 600 python scripts/role_cycles_rows.py v2:128,48,1,8192,0 v2:256,64,64,32768,0 mqa > gpurun_out/r03x/rc.jsonl 2> gpurun_out/r03x/rc.err
cat gpurun_out/r03x/rc.jsonl; tail -3 gpurun_out/r03x/rc.err
