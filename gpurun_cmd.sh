mkdir -p gpurun_out/p11
VISTA_LIB=$PWD/paper_2510_22049_b200/libvista_qt.so timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "softmax and not backward and not bwd or c5 or int8 or invariant or independence or smoke" > gpurun_out/p11/pytest_qt.log 2>&1; echo "pytest qt exit $?"; tail -2 gpurun_out/p11/pytest_qt.log
TAG=p11 VARIANTS="default qt" CFGS="c2 c3 c5" STEPS=100 bash scripts/ab_softmax.sh
TAG=p11b VARIANTS="qt default" CFGS="c2" STEPS=100 bash scripts/ab_softmax.sh
