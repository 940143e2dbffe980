mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
for DC in 1.25 1.4 1.6 1.8 2.0 2.4; do
  for cfg in mha7b_b16 mha7b_b32 gqa; do
    echo "DC=$DC $cfg $(BIFATTN_DEC_COST=$DC EXP_CFG=$cfg python scripts/exp_shapes.py 0,0 2>&1| cut -c1-60)"
  done
done 2>&1 | tee gpurun_out/deccost2.txt
