set -x
mkdir -p gpurun_out
timeout 600 python scripts/timeline.py mha7b_b32 mha7b_b32_fp8 mha7b_b16 > gpurun_out/timeline3.jsonl 2> gpurun_out/timeline3.err
