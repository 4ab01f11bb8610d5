python -m pytest tests/test_gpu_parity.py tests/test_gpu_config_scale.py tests/test_gpu_fused_sad.py tests/test_gpu_guards.py -k "sad or fused or guard" -x -q -p no:cacheprovider > gpurun_out/t20.log 2>&1; echo "tests rc=$?" >> gpurun_out/t20.log
python bench.py --config C2 --steps 200 --no-cpu-baseline --e2e-steps 2 > gpurun_out/s_c2.log 2>&1
MERIT_SAD_SPLIT=0 python bench.py --config C2 --steps 200 --no-cpu-baseline --e2e-steps 2 > gpurun_out/s_c2_nosplit.log 2>&1
python bench.py --no-cpu-baseline --e2e-steps 2 > gpurun_out/s_c5.log 2>&1
