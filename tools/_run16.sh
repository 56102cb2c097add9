timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pt16.log 2>&1
timeout 400 python bench.py --no-cpu --no-bootstrap > gpurun_out/bench16.log 2>&1
timeout 300 python tools/boot_bench.py 47 2 --graph > gpurun_out/boot16.log 2>&1
