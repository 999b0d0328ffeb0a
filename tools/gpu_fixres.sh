timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
python tools/sweep_config4.py > gpurun_out/sweep_c4.jsonl 2> gpurun_out/sweep_c4.err; echo sweep=$?
