DESC_LIB=build_variants/lib_trace_w2.so timeout 300 python scripts/scan_trace.py f32
for v in w1 w2 w3 w4 w2lb2; do for w in scan64M_f32 scan64M_i32; do
    if [ $v = base ]; then L=""; else L=build_variants/lib_$v.so; fi
    DESC_LIB=$L timeout 300 python bench.py --workload $w --scan-algo stream --no-oracle --steps 300 --warmup 20 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$w', d['value'], d['roofline']['frac'])"
done; done
