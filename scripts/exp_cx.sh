for L in trunc cx1 cx2 cx4 cx8 cx6 cx14; do
  for c in mqa gqa; do echo "$L $c $(EXP_LIB=exp_libs/$L.so EXP_CFG=$c timeout 60 python scripts/exp_shapes.py 8192,0 | cut -c1-80)"; done
done
