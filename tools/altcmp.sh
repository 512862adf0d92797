cd $GRAFT_REPO_ROOT
bash tools/ab_env.sh "QF_ALT=0 QF_ABLATE_ALT=1" "QF_ALT=1" 2 --layers 200
for A in 0 1; do
QF_ALT=$A timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_alt$A.csv python bench.py --steps 1 --warmup 0 --no-cpu --no-secondary --no-refsig --layers 40 > /dev/null 2>&1
done
