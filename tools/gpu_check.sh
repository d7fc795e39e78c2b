# GPU-side check used during development: the GPU test suite, then the
# reference's own suite (tools/ref_suite.py).  Logs land in gpurun_out/.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -q -rf -p no:cacheprovider --deselect tests/test_ref_suite.py ${PYTEST_ARGS:-} > gpurun_out/check_pytest.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/check_pytest.log
python tools/ref_suite.py run -- -q -rf > gpurun_out/check_refsuite.log 2>&1; echo "refsuite rc=$?"
tail -15 gpurun_out/check_refsuite.log
