timeout 900 python -m pytest tests/test_cli.py tests/test_cpp_facade.py -q 2>&1 | tail -25 > gpurun_out/r2_cli.log
