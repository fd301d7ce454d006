for cfg in "1 1e-2" "0 1e-2"; do
set -- $cfg
echo "== TC $1 REL_TOL32 $2"
MG_UPD_TC=$1 MG_REL_TOL32=$2 timeout 900 python tools/prof_embed.py --n 20000000 --stats 2>&1 | tail -5
done
