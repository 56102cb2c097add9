timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pt9.log 2>&1
timeout 300 python bench.py --no-cpu --no-bootstrap > gpurun_out/bench9.log 2>&1
LF_LIB_PATH=build/lib_pf.so timeout 300 python bench.py --no-cpu --no-bootstrap > gpurun_out/bench9pf.log 2>&1
timeout 300 python tools/boot_bench.py 47 2 --graph > gpurun_out/boot9.log 2>&1
LF_LIB_PATH=build/lib_pf.so timeout 300 python tools/boot_bench.py 47 2 --graph > gpurun_out/boot9pf.log 2>&1
