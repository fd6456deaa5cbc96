mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ordered.py -x -q > gpurun_out/r02c_ordered.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_ordered.py > gpurun_out/r02c_pytest.txt 2>&1
INET_B200_REFSUITE_LOG=gpurun_out/r02c_refsuite.txt timeout 1200 python -m pytest tests/test_reference_suite.py -q > gpurun_out/r02c_refsuite_outer.txt 2>&1
tail -3 gpurun_out/r02c_*.txt
