# the GPU test suite against the -DBIFATTN_CHECKS build (device-side bounds
# checks: a violation prints its line and traps) — the memory-safety evidence
# of round 3 while compute-sanitizer is closed on the pool
mkdir -p gpurun_out/r03checks
python -c "import __graft_entry__ as g; g.build(); from paper_2403_08845_b200 import _build; _build.build_variant('checks', ['-DBIFATTN_CHECKS'])" > /dev/null 2>&1
BIFATTN_TEST_LIB=$PWD/paper_2403_08845_b200/libbifattn_checks.so timeout -k 10 1200 python -m pytest tests -m gpu -q -x --timeout 300 -rA > gpurun_out/r03checks/pytest_gpu_checks.txt 2>&1
echo "exit $?" >> gpurun_out/r03checks/pytest_gpu_checks.txt
tail -3 gpurun_out/r03checks/pytest_gpu_checks.txt; grep -c "BA_CHECK failed" gpurun_out/r03checks/pytest_gpu_checks.txt
python - <<'PY'
import paper_2403_08845_b200 as ba, os
ba.load_library(os.path.join(os.getcwd(), "paper_2403_08845_b200/libbifattn_checks.so"))
print("checks library loaded:", ba._lib._name)
PY
