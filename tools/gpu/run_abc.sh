# A/B timing of K2 library variants on one box: tools/gpu/run_abc.sh "<libs>" "<shapes>" [J]
LIBS=${1:-"libautobyte.so"}; SHAPES=${2:-"3x256"}; J=${3:-4096}
for i in $(seq 1 ${ROUNDS:-2}); do
 for lib in $LIBS; do
  echo "== $lib"; AUTOBYTE_LIB=paper_2112_13509_b200/$lib timeout 300 python tools/kbench.py $J 64 64 $SHAPES 2>&1 | grep '^{'
 done
done
