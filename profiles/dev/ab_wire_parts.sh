# e2e of the host-call output wire, repeated (parts per slice A/B: build variants of
# kWirePartBytes into libbitmm_b200_<tag>.so.ab and list the tags in TAGS).
P=paper_2306_08960_b200
for v in ${TAGS:-cur cur cur}; do
  [ "$v" != cur ] && cp $P/libbitmm_b200_$v.so.ab $P/libbitmm_b200.so
  timeout 300 python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; e=json.load(sys.stdin)['e2e']; print('$v', round(e['value'],1), {k: round(v,3) for k,v in e['ms_per_call'].items()}, round(e['pageable_host_buffers']['value'],1))"
done
