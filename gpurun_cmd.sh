mkdir -p gpurun_out/p12
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "layers or smoke" > gpurun_out/p12/pytest.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/p12/pytest.log
TAG=p12 ENVS="VISTA_GEMM_PAIR=1;VISTA_GEMM_PAIR=0" CFGS="c2 c3" BARGS="--layers 3 --steps 10" bash scripts/ab_env.sh
