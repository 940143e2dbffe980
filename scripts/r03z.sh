mkdir -p gpurun_out/r03z
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout -k 10 900 python -m pytest tests -m gpu -q -x --timeout 120 -rA > gpurun_out/r03z/pytest_gpu.txt 2>&1
tail -2 gpurun_out/r03z/pytest_gpu.txt; grep -E "FAILED|Error|ap_rows|ap_dyn" gpurun_out/r03z/pytest_gpu.txt | head -12
