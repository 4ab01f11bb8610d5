timeout 300 python -m pytest tests/test_gpu_parity.py -k "conv_c3 or stride1 or conv_variants or device_buffers" -x -q -p no:cacheprovider > gpurun_out/t21.log 2>&1; echo "tests rc=$?" >> gpurun_out/t21.log
timeout 300 python -m pytest tests/test_gpu_config_scale.py -k "c3" -x -q -p no:cacheprovider >> gpurun_out/t21.log 2>&1; echo "tests2 rc=$?" >> gpurun_out/t21.log
timeout 300 python bench.py --config C3 --steps 200 --no-cpu-baseline --e2e-steps 2 > gpurun_out/p_c3.log 2>&1
MERIT_S1_PAIR=0 timeout 300 python bench.py --config C3 --steps 200 --no-cpu-baseline --e2e-steps 2 > gpurun_out/p_c3_single.log 2>&1
timeout 300 python bench.py --config C3 --steps 200 --no-cpu-baseline --e2e-steps 2 > gpurun_out/p_c3b.log 2>&1
