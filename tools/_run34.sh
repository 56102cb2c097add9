timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pt34.log 2>&1
for b in 1 8 32; do timeout 300 python bench.py --no-cpu --no-bootstrap --batch $b --steps 10 > gpurun_out/bb34_$b.log 2>&1; done
timeout 300 python tools/boot_bench.py 47 2 --graph --profile > gpurun_out/boot34.log 2>&1
