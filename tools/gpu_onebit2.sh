timeout 900 python -m pytest tests/test_gpu_onebit.py tests/test_gpu_exchange.py -q -k "onebit" 2>&1 | tail -3
python tools/prof_onebit_c3.py
bash tools/gpu_onebit_prof.sh 2>&1 | grep reduce_k
