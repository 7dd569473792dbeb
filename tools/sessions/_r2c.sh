set -u
bash tools/gpu_tests.sh r2c "multirank or c4_bench or tiny_corpus" 
bash tools/gpu_var.sh r2c "base=" "ev1=GML_EV_LOAD=1" "ev2=GML_EV_LOAD=2" "bfc2=GML_BFC_MINB=2" "bfc6=GML_BFC_MINB=6"
bash tools/gpu_sanitize.sh r2c
