cd $GRAFT_REPO_ROOT
for b in 18432 36864; do
 for m in 0 4 5 6; do ./scripts/mbf $b $m 4096 200 148 512 4; done
done
for m in 0 4 6; do ./scripts/mbf 18432 $m 4096 200 148 512 2; done
