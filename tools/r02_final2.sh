#!/bin/bash
# round-2 closing run: GPU suite, smoke, default bench (timed), reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fin2_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/fin2_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin2_smoke.log 2>&1
t0=$(date +%s); timeout 900 python bench.py > gpurun_out/fin2_bench.json 2> gpurun_out/fin2_bench.err; t1=$(date +%s); echo "bench wall $((t1-t0)) s" >> gpurun_out/fin2_bench.err
t0=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/fin2_ref.json 2> gpurun_out/fin2_ref.err; t1=$(date +%s); echo "ref wall $((t1-t0)) s" >> gpurun_out/fin2_ref.err
echo done
