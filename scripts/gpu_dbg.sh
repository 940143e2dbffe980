for c in mha7b_b32 mha7b_b16; do
for d in 1 128 256; do
  echo "$c dbg=$d $(BIFATTN_DBG=$d timeout 120 python scripts/exp_ab.py $c 2>&1 | tail -1)"
done; done
