mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
for cfg in mha7b_b16 mha7b_b32 gqa mqa long; do
  echo "default $cfg $(EXP_CFG=$cfg python scripts/exp_shapes.py 0,0 2>&1| cut -c1-70)"
done
for DC in 3.0 3.5 4.5; do
  echo "DC=$DC mqa $(BIFATTN_DEC_COST=$DC EXP_CFG=mqa python scripts/exp_shapes.py 0,0 2>&1| cut -c1-70)"
done
python scripts/bench_multitoken.py 2>&1 | cut -c1-150
