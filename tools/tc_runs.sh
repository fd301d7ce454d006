timeout 300 python tools/bench_update.py 2000000 20000000 2>&1 | grep "variant 1"
for d in 4 6; do echo "== dbg $d"; MG_U3_DBG=$d timeout 300 python tools/bench_update.py 20000000 2>&1 | grep "variant 1"; done
for rt in 1e-2 3e-2; do
echo "== TC 1 REL_TOL32 $rt"
MG_UPD_TC=1 MG_REL_TOL32=$rt timeout 300 python tools/prof_embed.py --n 2000000 --stats 2>&1 | tail -5
done
