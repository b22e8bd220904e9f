mkdir -p gpurun_out/p10
VISTA_SOFTMAX_CMAX=2 timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "softmax or c5 or int8 or partial or invariant or independence" > gpurun_out/p10/pytest_cmax2.log 2>&1; echo "pytest cmax2 exit $?"; tail -2 gpurun_out/p10/pytest_cmax2.log
TAG=p10 VARIANTS="default prev" CFGS="c2 c5" STEPS=100 bash scripts/ab_softmax.sh
TAG=p10 ENVS="VISTA_SOFTMAX_CMAX=2;VISTA_SOFTMAX_CMAX=8" CFGS="c5" REPS=2 bash scripts/ab_env.sh
TAG=p10b VARIANTS="prev default" CFGS="c2" STEPS=100 bash scripts/ab_softmax.sh
