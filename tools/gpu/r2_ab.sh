DYNRAD_LIB=variants/trace0.so timeout 300 python tools/trace_pp.py
for rep in 1 2; do
  for v in pp db rp; do DYNRAD_K6=$v TAG=$v timeout 300 python tools/ab_k6.py; done
  DYNRAD_LIB=variants/p1111.so TAG=pp_p1111 timeout 300 python tools/ab_k6.py
done
