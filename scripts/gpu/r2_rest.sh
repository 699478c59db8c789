python -c "import __graft_entry__ as g; g.build()" || exit 1
g++ -std=c++20 -O2 -Wall -Iinclude tests/cpp/test_api.cpp -Lpaper_2509_09139_b200/lib -lhpbj -Wl,-rpath,$PWD/paper_2509_09139_b200/lib -o /tmp/test_api && timeout 300 /tmp/test_api > gpurun_out/r2_test_api.log 2>&1; echo "rc=$?" >> gpurun_out/r2_test_api.log
timeout 1800 python -X faulthandler -m pytest tests -m gpu -v -rA -p no:cacheprovider --deselect tests/test_gpu_kernels.py --deselect tests/test_gpu_solve.py::test_config4_newton_sequence --deselect tests/test_gpu_solve.py::test_large_config_solve > gpurun_out/r2_pytest_rest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest_rest.log
