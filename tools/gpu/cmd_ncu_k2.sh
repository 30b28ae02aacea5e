# one ncu --set full capture of K2 at the given shape (default 3x256, J = 1024 jobs x 4096 candidates)
SHAPE=${1:-3x256}; J=${2:-1024}; TAG=${3:-k2}
python tools/kbench.py $J 64 64 $SHAPE > gpurun_out/${TAG}_pre.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 2 -c 1 -o gpurun_out/${TAG} python tools/kbench.py $J 64 64 $SHAPE > gpurun_out/${TAG}_ncu.log 2>&1
ncu -i gpurun_out/${TAG}.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv
ncu -i gpurun_out/${TAG}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_src.csv 2>/dev/null
ncu -i gpurun_out/${TAG}.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv
