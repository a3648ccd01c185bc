T="tests/test_gpu_parity.py::test_contraction_path"
for pre in "tests/test_epilogue.py" "tests/test_benched_parity.py" "tests/test_abi.py tests/test_bench_multirank.py" "tests/test_cli.py" "tests/test_gpu_parity.py::test_generic_bit_exact_random tests/test_gpu_parity.py::test_default_plans_random tests/test_gpu_parity.py::test_gett_random_two_operand"; do
  timeout 300 python -m pytest $pre $T -m gpu -x -q -p no:cacheprovider > /tmp/b.log 2>&1; echo "pre=[$pre] rc=$?"; tail -1 /tmp/b.log
done
