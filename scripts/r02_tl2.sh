set -x
mkdir -p gpurun_out
timeout -k 10 600 python scripts/timeline.py mha7b_b32 mha7b_b32_fp8 mha7b_b16 > gpurun_out/timeline11.jsonl 2> gpurun_out/timeline11.err
