mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multitoken.py -q -x --timeout 60 2>&1 | tail -2
python scripts/exp_ab_lib.py exp_libs/prev.so exp_libs/trunc.so
for c in mqa gqa long; do echo "$c $(EXP_CFG=$c timeout 120 python scripts/exp_shapes.py 0,0 | cut -c1-90)"; done
