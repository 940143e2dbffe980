set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
# knob sweeps on an experiment build (release builds ignore the environment)
BIFATTN_NPB=2 timeout -k 10 600 python scripts/ab.py mha7b_b32 3 exp -DBIFATTN_EXPERIMENTS > gpurun_out/ab_npb2.json 2> gpurun_out/ab3.err
BIFATTN_DEC_COST=1.6 timeout -k 10 600 python scripts/ab.py mha7b_b32 3 exp -DBIFATTN_EXPERIMENTS > gpurun_out/ab_dc16.json 2>> gpurun_out/ab3.err
BIFATTN_DEC_COST=1.25 timeout -k 10 600 python scripts/ab.py mha7b_b32 3 exp -DBIFATTN_EXPERIMENTS > gpurun_out/ab_dc125.json 2>> gpurun_out/ab3.err
BIFATTN_SWG=4 timeout -k 10 600 python scripts/ab.py mha7b_b32 3 exp -DBIFATTN_EXPERIMENTS > gpurun_out/ab_swg4.json 2>> gpurun_out/ab3.err
BIFATTN_SEG_PENALTY=4 timeout -k 10 600 python scripts/ab.py mha7b_b32 3 exp -DBIFATTN_EXPERIMENTS > gpurun_out/ab_seg4.json 2>> gpurun_out/ab3.err
BIFATTN_DEC_COST=1.5 timeout -k 10 600 python scripts/ab.py mha7b_b32_fp8 3 exp -DBIFATTN_EXPERIMENTS > gpurun_out/ab_fp8_dc15.json 2>> gpurun_out/ab3.err
BIFATTN_DEC_COST=1.9 timeout -k 10 600 python scripts/ab.py mha7b_b32_fp8 3 exp -DBIFATTN_EXPERIMENTS > gpurun_out/ab_fp8_dc19.json 2>> gpurun_out/ab3.err
