cd $GRAFT_REPO_ROOT
for b in 1 2; do (cd .ab/$b && python paper_1912_06680_b200/build.py > /dev/null 2>&1); done
for i in 1 2 3; do for b in 1 2; do echo "build $b ($(cat .ab/$b/REV))" >> gpurun_out/r2_loss_ab.txt; timeout 300 python tools/loss_probe.py --lib-root .ab/$b --reps 50 >> gpurun_out/r2_loss_ab.txt 2>&1; done; done
echo done
