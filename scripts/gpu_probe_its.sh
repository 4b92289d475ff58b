cd $GRAFT_REPO_ROOT
for cfg in c3 c1 c2; do for its in 48 16 8; do
 RSM_EIG_PROBE_ITS=$its REPS=7 timeout 300 python scripts/prof_c3.py $cfg > /tmp/o.log 2>&1
 echo "$cfg its=$its $(grep median /tmp/o.log) $(tail -2 /tmp/o.log | head -1 | grep -o "'matvecs': [0-9.]*")"
done; done
