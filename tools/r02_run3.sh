mkdir -p gpurun_out/r3
timeout -s KILL 900 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_certificate.py -q -s -p no:cacheprovider > gpurun_out/r3/pytest_sharded_cert.txt 2>&1; grep -E "worst|passed|failed|FAILED|Error" gpurun_out/r3/pytest_sharded_cert.txt | head -40
timeout -s KILL 1800 python -m pytest tests/test_gpu_fullsize.py -q -s -p no:cacheprovider --durations=0 > gpurun_out/r3/pytest_fullsize.txt 2>&1; grep -E "checked|passed|failed|FAILED|Error|s call" gpurun_out/r3/pytest_fullsize.txt | head -40
