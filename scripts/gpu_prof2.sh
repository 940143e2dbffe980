mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
( EXP_LIB=exp_libs/prof.so python scripts/exp_prof.py mha7b_b32 | head -20
  EXP_LIB=exp_libs/prof.so EXP_MC=16384 EXP_MD=0 python scripts/exp_prof.py gqa | head -20
  EXP_LIB=exp_libs/prof.so EXP_MC=16384 EXP_MD=0 BIFATTN_N=16 python scripts/exp_prof.py gqa | head -20
) 2>&1 | tee gpurun_out/prof2.txt
