set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.txt 2>&1
timeout -k 10 900 python scripts/ab.py mha7b_b32 3 nonarrow -DBIFATTN_NO_NARROW > gpurun_out/ab_narrow_b32.json 2> gpurun_out/ab_narrow.err
timeout -k 10 600 python scripts/ab.py mha7b_b16 3 nonarrow -DBIFATTN_NO_NARROW > gpurun_out/ab_narrow_b16.json 2>> gpurun_out/ab_narrow.err
