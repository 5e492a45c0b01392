run() { echo "== $*"; env "$@" python tools/optime.py $CFG 2>&1 | tail -4; }
for CFG in 2 3; do
run A=base
run RQ_TILE_LEAVES=192
run RQ_TILE_LEAVES=256
run RQ_TILE_LEAVES=384
run RQ_TILE_LEAVES=512
done
