# planner weights: decode-tile cost and segment penalty (product build)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
for DC in 0.8 0.9 1.0 1.1 1.25 1.4; do
  for cfg in mha7b_b32 mha7b_b16; do
    echo "DC=$DC $cfg $(BIFATTN_DEC_COST=$DC EXP_CFG=$cfg python scripts/exp_shapes.py 8192,256 | cut -c1-60)"
  done
done 2>&1 | tee gpurun_out/deccost.txt
for SP in 0 1 2 4 8; do
  echo "SP=$SP $(BIFATTN_SEG_PENALTY=$SP EXP_CFG=mha7b_b32 python scripts/exp_shapes.py 8192,256 | cut -c1-60)"
done 2>&1 | tee -a gpurun_out/deccost.txt
