mkdir -p gpurun_out
timeout 300 python tools/prof_codec.py --case mlp --iters 200
