set -u
ARROW_C5_SAMPLE=16384 bash scripts/ab_c5.sh build/ab/cur4.so build/ab/ptx_o1.so build/ab/cicc_o2.so
