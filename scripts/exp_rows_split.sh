mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
for NS in 0 2 3 6; do
 for c in mqa gqa long; do
  echo "NS=$NS $c $(BIFATTN_ROWS_SPLITS=$NS BIFATTN_CTX_ROWS=2 EXP_CFG=$c timeout 120 python scripts/exp_shapes.py 0,0 | cut -c1-130)"
 done
done
