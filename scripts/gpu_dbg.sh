for L in exp_libs/exp.so paper_2403_08845_b200/libbifattn.so; do echo "$L $(EXP_LIB=$L python scripts/exp_graph.py 1280,0 8192,256 2>&1 | tail -2 | tr '\n' ' ' | sed 's/"host_us_per_call"[^,]*,//g')"; done
echo "b16 $(timeout 120 python scripts/exp_ab.py mha7b_b16 2>&1 | tail -1)"
echo "b32 $(timeout 120 python scripts/exp_ab.py mha7b_b32 2>&1 | tail -1)"
python scripts/exp_shapes.py 128,512 8192,0 2>&1 | cut -c1-90
