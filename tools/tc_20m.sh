for d in 1 0; do
echo "== DERIVE $d"
MG_GRAM_DERIVE=$d timeout 900 python tools/prof_embed.py --n 20000000 --stats 2>&1 | tail -5
done
