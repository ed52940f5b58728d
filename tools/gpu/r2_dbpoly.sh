for rep in 1 2; do
  DYNRAD_K6=db TAG=db timeout 300 python tools/ab_k6.py
  for m in 01 11 55; do DYNRAD_K6=db DYNRAD_LIB=variants/db$m.so TAG=db$m timeout 300 python tools/ab_k6.py; done
done
