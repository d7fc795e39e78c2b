for L in 128 256 512; do QADIC_TZ_L=$L python tools/ab/polylong_scale.py 2>&1 | grep "d=1.*auto" | sed "s/^/TL=$L /"; done
QADIC_TZ_L=128 python -m pytest tests/test_gpu_domain.py -m gpu -x -q -p no:cacheprovider -k "long" 2>&1 | tail -1
