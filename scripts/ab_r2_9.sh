set -u
ROUNDS=2 bash scripts/ab.sh build/ab/cur4.so build/ab/lat3.so build/ab/lat4.so
