# same-box A/B of two libraries on the C4 bench line (interleaved, 2 rounds)
for i in 1 2; do for lib in $1 $2; do
  AUTOBYTE_LIB=paper_2112_13509_b200/$lib timeout 300 python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('$lib', round(d['value']/1e6,1), round(d['roofline']['frac'],4), round(d['per_kernel_ms']['score_ms'],3), d['clocks']['sm_mhz'])"
done; done
