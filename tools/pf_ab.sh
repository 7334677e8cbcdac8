# L2 prefetch warp A/B at C1, C2 and C4 (decode tok/s): bash tools/pf_ab.sh "ENV=..." ...
for v in "$@"; do
  echo "== $v"
  env $v timeout 200 python tools/c1_grid.py
  env $v timeout 300 python tools/c4_decode.py | tail -2
done
