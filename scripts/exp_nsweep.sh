# chunk width N sweep per config, decomposed into decode-only / context-only / full shapes
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
for N in 16 32 64; do
  echo "== long N=$N"; BIFATTN_N=$N EXP_CFG=long timeout 300 python scripts/exp_shapes.py 128,1024 32768,0 32768,1024
  echo "== gqa N=$N"; BIFATTN_N=$N EXP_CFG=gqa timeout 300 python scripts/exp_shapes.py 128,512 16384,0 16384,512
  echo "== b32 N=$N"; BIFATTN_N=$N EXP_CFG=mha7b_b32 timeout 300 python scripts/exp_shapes.py 128,256 8192,0 8192,256
done 2>&1 | tee gpurun_out/nsweep.txt
