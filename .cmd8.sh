python tools/measure_probe.py > gpurun_out/m8.log 2>&1
MERIT_PDL=0 python tools/measure_probe.py > gpurun_out/m8_nopdl.log 2>&1
