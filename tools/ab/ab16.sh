python -m pytest tests/test_gpu_domain.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "long or fqt or polymul" > gpurun_out/ab16_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ab16_pytest.log
python tools/ab/polylong_scale.py 2>&1 | grep auto
QADIC_TZ_MATERIALIZE=1 python tools/ab/polylong_scale.py 2>&1 | grep auto | sed 's/^/MAT /'
