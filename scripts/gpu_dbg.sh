timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x 2>&1 | tail -2
for L in exp_libs/HEAD.so paper_2403_08845_b200/libbifattn.so; do
echo "$L"; EXP_LIB=$L python scripts/exp_shapes.py 128,512 8192,256 8192,0 2>&1 | cut -c1-90
echo "b16 $(EXP_LIB=$L timeout 120 python scripts/exp_ab.py mha7b_b16 2>&1 | tail -1)"
done
