bash tools/icache_lib.sh ablibs/cur.so ablibs/b6.so ablibs/b5.so
python tools/ab.py ablibs/cur.so ablibs/b6.so ablibs/b5.so --reps 2 --only c3,c4
for S in 2 5 8; do echo "slack $S"; MCSG_DEBUG_COMPACT_SLACK=$S python tools/ab.py ablibs/cur.so --reps 1 --only c3,c4; done
