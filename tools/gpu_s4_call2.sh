O=gpurun_out
python tools/c4_geo_ab.py > $O/s4_geo_ab.log 2>&1
timeout 900 python -m pytest tests/test_gpu_bench_paths.py tests/test_gpu_parity.py tests/test_gpu_features.py -q -x > $O/s4_geo_tests.log 2>&1; echo "rc=$?" >> $O/s4_geo_tests.log
