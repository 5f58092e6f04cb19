cd $GRAFT_REPO_ROOT
for cfg in "2 0 8" "2 8 8" "2 2 8" "2 1 8" "2 1 12" "2 0 12" "1 0 8" "0 0 8"; do
set -- $cfg
echo "sched $1 syncj $2 group $3"; XTSG_TTM_SCHED=$1 XTSG_TTM_SYNCJ=$2 XTSG_TTM_GROUP=$3 timeout 300 python tools/c3_compress_probe.py 400
done
