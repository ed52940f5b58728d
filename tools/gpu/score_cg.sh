for cg in "" 1 2 4; do
  if [ -z "$cg" ]; then E=""; else E="DYNRAD_SCORE_CG=$cg"; fi
  echo "== CG $cg"; env $E timeout 200 python tools/dyn_stats.py | grep hunyuan | grep -o "build ms.*"
  env $E timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:score_kernel -c 2 python tools/dyn_stats.py 2>/dev/null | grep -E "score_kernel|duration" | paste - - | awk '{print $2, $3, $(NF)}'
done
