./tools/probes/tc_probe > gpurun_out/r02_tc_probe.log 2>&1; echo rc=$? >> gpurun_out/r02_tc_probe.log
python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest_d.log 2>&1; echo rc=$? >> gpurun_out/r02_gputest_d.log
