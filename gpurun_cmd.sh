mkdir -p gpurun_out/p6
TAG=p6 VARIANTS="default v33 r8 fakeexp v33fake" CFGS="c2 c5" STEPS=100 bash scripts/ab_softmax.sh
TAG=p6 VARIANTS="v33 default" CFGS="c2 c3" STEPS=100 bash scripts/ab_softmax.sh
