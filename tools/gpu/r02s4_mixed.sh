timeout 900 python -c "
import bench, json
m = bench.mixed_trace()
print(json.dumps({k: v for k, v in m.items() if k != 'ranks'}))
print(json.dumps(m['ranks'][0]))
"
