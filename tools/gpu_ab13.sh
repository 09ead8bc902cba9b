V='[{"mode":"f32","config":1},{"mode":"f32","config":8},{"mode":"f32","config":6},{"mode":"f16","config":1},{"mode":"f16","config":8},{"mode":"f16","config":6}]'
for sh in "8192 8192 8192" "16384 16384 16384" "4096 4096 4096" "8192 4096 4096" "16384 4096 1024" "32768 1024 4096"; do set -- $sh; M=$1 N=$2 K=$3 VARIANTS="$V" ROUNDS=5 REPS=$((2000000000000 / ($1*$2*$3) + 3)) python tools/ab.py; done
