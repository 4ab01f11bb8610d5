python -m pytest tests/test_gpu_measured_traffic.py tests/test_cpp_dropin.py -x -q -s -p no:cacheprovider > gpurun_out/t7.log 2>&1; echo "tests rc=$?" >> gpurun_out/t7.log
