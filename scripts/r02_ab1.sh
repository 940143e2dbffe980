set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout -k 10 900 python scripts/ab.py mha7b_b32 4 nopf -DBIFATTN_NO_L2PF > gpurun_out/ab_pf_b32.json 2> gpurun_out/ab_pf.err
timeout -k 10 600 python scripts/ab.py mha7b_b16 3 nopf -DBIFATTN_NO_L2PF > gpurun_out/ab_pf_b16.json 2>> gpurun_out/ab_pf.err
timeout -k 10 600 python scripts/timeline.py mha7b_b32 mha7b_b32_fp8 > gpurun_out/timeline7.jsonl 2> gpurun_out/timeline7.err
