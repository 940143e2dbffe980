for r in 1 2; do for c in mha7b_b32 mha7b_b16; do
  echo "head $(EXP_LIB=exp_libs/head.so timeout 120 python scripts/exp_ab.py $c 2>&1 | tail -1)"
  echo "cur  $(timeout 120 python scripts/exp_ab.py $c 2>&1 | tail -1)"
done; done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
