mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
for cfg in mha7b_b16 mha7b_b32 gqa mqa long; do
  echo "default $cfg $(EXP_CFG=$cfg python scripts/exp_shapes.py 0,0 2>&1| cut -c1-70)"
done
for DC in 1.25 2.0 2.6; do
  for cfg in mqa long; do
    echo "DC=$DC $cfg $(BIFATTN_DEC_COST=$DC EXP_CFG=$cfg python scripts/exp_shapes.py 0,0 2>&1| cut -c1-70)"
  done
done
for DC in 1.25 2.0 2.6; do
  echo "DC=$DC b32 n4 $(BIFATTN_DEC_COST=$DC python scripts/bench_multitoken.py 2>&1 | grep '"n_tok": 4' | cut -c1-90)"
done
echo "default b32 n4 $(python scripts/bench_multitoken.py 2>&1 | grep '"n_tok": 4' | cut -c1-90)"
