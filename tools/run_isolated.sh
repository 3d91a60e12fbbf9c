#!/bin/bash
# Run each selected pytest node in its own process under a timeout (a hung kernel cannot stall the rest).
#   tools/run_isolated.sh <timeout_s> <pytest -k expr> [test files...]
T=$1; K=$2; shift 2
FILES=${@:-tests}
for id in $(python -m pytest $FILES --collect-only -q -k "$K" 2>/dev/null | grep "::"); do
  out=$(timeout $T python -m pytest "$id" -x -q 2>&1)
  rc=$?
  if [ $rc -eq 0 ]; then echo "PASS $id"; elif [ $rc -eq 124 ]; then echo "TIMEOUT $id"; else
    echo "FAIL $id"; echo "$out" | grep -E "^E |Error|assert" | head -8; fi
done
