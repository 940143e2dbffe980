set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout -k 10 900 python -m pytest tests -m gpu -q -x --timeout 60 > gpurun_out/pytest_gpu.txt 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu.txt
timeout -k 10 900 python scripts/ab.py mha7b_b32 3 nopool -DBIFATTN_NO_POOL > gpurun_out/ab_pool_b32.json 2> gpurun_out/ab_pool.err
timeout -k 10 600 python scripts/ab.py mha7b_b16 3 nopool -DBIFATTN_NO_POOL > gpurun_out/ab_pool_b16.json 2>> gpurun_out/ab_pool.err
timeout -k 10 600 python scripts/ab.py mha7b_b32_fp8 3 nopool -DBIFATTN_NO_POOL > gpurun_out/ab_pool_fp8.json 2>> gpurun_out/ab_pool.err
timeout -k 10 600 python scripts/timeline.py mha7b_b32 > gpurun_out/timeline10.jsonl 2> gpurun_out/timeline10.err
