python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "u64 or LayerK" > gpurun_out/ab7_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/ab7_pytest.log
python tools/mm64_profile.py; python tools/mm64_profile.py | head -1
timeout 300 python bench.py --config mm64 > gpurun_out/ab7_mm64.json 2>&1; tail -c 400 gpurun_out/ab7_mm64.json
