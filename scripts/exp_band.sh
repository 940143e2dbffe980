# context band width sweep (BIFATTN_BAND) on the configs with several row chunks
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt
for B in 4 8 16 32 9999; do
  echo "== band $B"
  BIFATTN_BAND=$B EXP_CFG=gqa timeout 300 python scripts/exp_shapes.py 16384,0 16384,512
  BIFATTN_BAND=$B EXP_CFG=long timeout 300 python scripts/exp_shapes.py 32768,0 32768,1024
  BIFATTN_BAND=$B EXP_CFG=mqa timeout 300 python scripts/exp_shapes.py 8192,256
  BIFATTN_BAND=$B timeout 300 python scripts/bench_multitoken.py | grep '"n_tok": 4'
done 2>&1 | tee gpurun_out/band.txt
