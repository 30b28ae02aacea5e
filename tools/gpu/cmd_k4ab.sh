# K4 A/B: adapt_bench at several (L, H, B) for two libraries, interleaved, 2 rounds
for i in 1 2; do for lib in $1 $2; do for cfg in "4 512 1024" "4 512 4096" "3 256 256" "4 512 100" "3 256 8192"; do
  AUTOBYTE_LIB=paper_2112_13509_b200/$lib timeout 120 python tools/adapt_bench.py $cfg 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('$lib', d['L'], d['H'], d['B'], round(d['adapt_ms']*1e3,1), 'us')"
done; done; done
