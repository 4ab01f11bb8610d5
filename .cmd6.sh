python -m pytest tests/test_gpu_parity.py tests/test_gpu_config_scale.py tests/test_gpu_fused_sad.py tests/test_gpu_guards.py -k "sad or fused or guard" -x -q -p no:cacheprovider > gpurun_out/t6.log 2>&1; echo "tests rc=$?" >> gpurun_out/t6.log
python bench.py --config C2 --steps 200 --no-cpu-baseline > gpurun_out/b6_c2.log 2>&1
python bench.py --no-cpu-baseline > gpurun_out/b6_c5.log 2>&1
python bench.py --no-cpu-baseline --no-fuse > gpurun_out/b6_c5sep.log 2>&1
python bench.py --config C3 --steps 200 --no-cpu-baseline > gpurun_out/b6_c3.log 2>&1
