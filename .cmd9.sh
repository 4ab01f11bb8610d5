MERIT_MEASURE_SELFTEST=1 python tools/measure_probe.py > gpurun_out/m9.log 2>&1
