#!/bin/bash
# GPU verification (run under gpurun): build, all GPU tests, smoke, bench line.  usage: tools/gpu_verify.sh <tag>
tag=${1:-ver}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || { echo build failed; tail gpurun_out/${tag}_build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_gpu_tests.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/${tag}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/${tag}_smoke.log
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"
cut -c1-700 gpurun_out/${tag}_bench.json
