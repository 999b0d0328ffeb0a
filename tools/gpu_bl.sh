timeout 900 python -m pytest tests/test_blocked.py -m gpu -x -q 2>&1 | tail -1
python tools/prof_blocked.py > gpurun_out/blocked.jsonl; python -c "
import json
for l in open('gpurun_out/blocked.jsonl'):
    r=json.loads(l); print(r['log2'], r['block'], round(r['encode_us'],1), round(r['encode_GBps']), round(r['decode_us'],1), round(r['decode_GBps']))"
