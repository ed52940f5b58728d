mkdir -p gpurun_out
run() { echo "== $1"; shift; env "$@" timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:score_kernel -c 2 --csv python tools/dyn_stats.py 2>/dev/null | grep score_kernel | awk -F'","' '{print $5, $NF}' | cut -c1-120; }
run base X=1
run base_cg2 DYNRAD_SCORE_CG=2
run abl1_noepi DYNRAD_LIB=$PWD/variants/msabl1.so
run abl2_nomma DYNRAD_LIB=$PWD/variants/msabl2.so
run abl2_nomma_cg2 DYNRAD_LIB=$PWD/variants/msabl2.so DYNRAD_SCORE_CG=2
run abl1_noepi_cg2 DYNRAD_LIB=$PWD/variants/msabl1.so DYNRAD_SCORE_CG=2
