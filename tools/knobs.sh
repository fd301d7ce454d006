for tc in 0 1; do
for rt in 1e-2 3e-2 1e-1; do
for ft in 1e-4 1e-3 1e-2; do
echo "== TC $tc REL_TOL32 $rt FAST_TOL32 $ft"
MG_UPD_TC=$tc MG_REL_TOL32=$rt MG_FAST_TOL32=$ft timeout 300 python tools/prof_embed.py --n 2000000 2>&1 | grep "^rep"
done; done; done
