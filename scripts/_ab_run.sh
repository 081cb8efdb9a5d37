for v in "" s2nl2 s2nl4; do
  MFADD_LIB_VARIANT=$v python scripts/kernel_times.py --config C5 --tag "s2-$v"
  MFADD_LIB_VARIANT=$v python scripts/time_solve.py --config C5 --tag "s2-$v"
  MFADD_LIB_VARIANT=$v python scripts/time_solve.py --config C2 --tag "s2-$v"
done
MFADD_LIB_VARIANT=s2nl2 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py -m gpu -x -q 2>&1 | tail -2
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python scripts/time_solve.py --config C4; python scripts/time_solve.py --config C3
