run() { echo "== $*"; env "$@" python tools/optime.py 2 2>&1 | tail -3; }
run A=base
run RQ_LIB_PATH=$PWD/exp/librigidq_skipmath.so
run RQ_LIB_PATH=$PWD/exp/librigidq_skipmath.so RQ_WAVE_THREADS=96 RQ_WAVE_CAPS=32,32,32,10240,96,384,72
