#!/bin/bash
# round-2 evidence: GPU suite, smoke, default bench, ncu launch list of the bench
# command, ncu --set full of the dominant kernel (balanced backward pass)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fin_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/fin_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-secondary --no-refsig > gpurun_out/fin_ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pass_bwd_dual --launch-skip 10 -c 1 -o gpurun_out/fin_bwd -f python bench.py --steps 1 --warmup 0 --no-cpu --no-secondary --no-refsig --layers 20 > gpurun_out/fin_ncu_bwd.log 2>&1
echo done
