# A/B of the pair kernel's in-slice lane barrier spacing at C3 (XTSG_TTM_SYNCJ:
# 0 = once per slice, n = every n j tiles), alternating, then one ncu capture
# of a current-build C3 TTM launch.
cd ${GRAFT_REPO_ROOT:-.}
for rep in 1 2 3; do for sj in 0 2 1 4; do
echo "syncj $sj rep $rep"; XTSG_TTM_SYNCJ=$sj timeout 300 python tools/c3_compress_probe.py 800
done; done
