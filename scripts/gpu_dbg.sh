python scripts/exp_sets.py mha7b_b32 8
python scripts/exp_sets.py mha7b_b32 8
