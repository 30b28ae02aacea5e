# one ncu --set full capture of K4 (adapt_kernel) at (L, H, B) with the source view exported
L=${1:-4}; H=${2:-512}; B=${3:-1024}; TAG=${4:-k4}
python tools/adapt_bench.py $L $H $B > gpurun_out/${TAG}_pre.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:adapt_kernel -s 2 -c 1 -o gpurun_out/${TAG} python tools/adapt_bench.py $L $H $B --once > gpurun_out/${TAG}_ncu.log 2>&1
ncu -i gpurun_out/${TAG}.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv
ncu -i gpurun_out/${TAG}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_src.csv 2>/dev/null
