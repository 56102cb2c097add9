timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pt22.log 2>&1
timeout 300 python tools/boot_bench.py 47 2 --graph --profile > gpurun_out/boot22.log 2>&1
