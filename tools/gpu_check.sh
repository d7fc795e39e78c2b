set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -q -rf -p no:cacheprovider --deselect tests/test_ref_suite.py > gpurun_out/check_pytest.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/check_pytest.log
python tools/ref_suite.py run -- -q -rf > gpurun_out/check_refsuite.log 2>&1; echo "refsuite rc=$?"
tail -40 gpurun_out/check_refsuite.log
