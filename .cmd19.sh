V=$PWD/paper_1911_03458_b200/variants
MERIT_DEV_LIB=$V/libmerit_dev_jouter.so python bench.py --no-cpu-baseline --e2e-steps 2 > gpurun_out/v_jouter.log 2>&1
python bench.py --no-cpu-baseline --e2e-steps 2 > gpurun_out/v_base3.log 2>&1
MERIT_DEV_LIB=$V/libmerit_dev_jouter.so python -m pytest tests/test_gpu_fused_sad.py -x -q -k "not c5" > gpurun_out/v_jouter_t.log 2>&1
