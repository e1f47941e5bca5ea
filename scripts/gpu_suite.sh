#!/bin/bash
# Full GPU pass: pytest -m gpu, smoke, bench.  Output under gpurun_out/$1.
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-suite}
mkdir -p $O
timeout 3000 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1
echo "pytest rc=$?" > $O/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/rc.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
echo "bench rc=$?" >> $O/rc.txt
