python tools/lmp_build_bench.py C4 256 2>&1 | grep -v Warn
WC4DVAR_GEMM_SYRK=0 python tools/lmp_build_bench.py C4 256 revd 2>&1 | grep -v Warn
python tools/lmp_build_bench.py C2 100 2>&1 | grep -v Warn
timeout 1500 python -m pytest tests/test_gpu_algorithms.py tests/test_gpu_distributed.py tests/test_gpu_rank.py tests/test_gpu_acceptance.py tests/test_gpu_configs_parity.py -q -x -k "not c2_inner" 2>&1 | tail -3
