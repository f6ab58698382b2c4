set -u
ARROW_C5_SAMPLE=16384 bash scripts/ab_c5.sh build/ab/cur3.so build/ab/cur3_tp4.so build/ab/cur3_tp2.so
