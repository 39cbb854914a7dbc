P="0.05:10 0.01:20 0.02:10"
echo "== lean"; timeout 600 python tools/sweep_counters.py 1.3e9 $P 2>&1 | cut -c1-70
echo "== tile"; MA_TILE=1 timeout 600 python tools/sweep_counters.py 1.3e9 $P 2>&1 | cut -c1-70
echo "== fastcta"; MA_FAST_CTA=1 timeout 600 python tools/sweep_counters.py 1.3e9 $P 2>&1 | cut -c1-70
echo "== warpexact"; MA_WARP_EXACT=1 timeout 600 python tools/sweep_counters.py 1.3e9 $P 2>&1 | cut -c1-70
