python -m pytest tests/test_gpu_domain.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "long or fqt or polymul" > gpurun_out/ab18_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/ab18_pytest.log
python tools/ab/polylong_scale.py 2>&1 | grep auto
python tools/ab/polylong_prof.py 1024
python tools/ab/polylong_prof.py 16; QADIC_CONV_PAIR=0 python tools/ab/polylong_scale.py 2>&1 | grep "d=1.*auto" | sed "s/^/NOPAIR /"
