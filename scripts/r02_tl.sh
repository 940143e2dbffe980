set -x
mkdir -p gpurun_out
timeout -k 10 600 python scripts/timeline.py mha7b_b32 mha7b_b32_fp8 > gpurun_out/timeline9.jsonl 2> gpurun_out/timeline9.err
