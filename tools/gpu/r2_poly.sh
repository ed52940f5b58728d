for lib in trace0 trace5555; do echo "== $lib"; DYNRAD_LIB=variants/$lib.so timeout 300 python tools/trace_pp.py; done
for rep in 1 2; do
  TAG=base timeout 300 python tools/ab_k6.py
  for m in 1111 2525 5555 b5b5; do DYNRAD_LIB=variants/p$m.so TAG=p$m timeout 300 python tools/ab_k6.py; done
  DYNRAD_K6=db TAG=db timeout 300 python tools/ab_k6.py
done
