timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x 2>&1 | tail -2
for L in exp_libs/HEAD.so paper_2403_08845_b200/libbifattn.so; do echo "$L"; EXP_LIB=$L python scripts/exp_graph.py 8192,256 128,512 2>&1 | tail -2; done
echo "b16 $(timeout 120 python scripts/exp_ab.py mha7b_b16 2>&1 | tail -1)"
