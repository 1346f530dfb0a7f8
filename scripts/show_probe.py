import ast
import sys

for line in open(sys.argv[1]):
    if line.startswith('{'):
        continue
    if not line.startswith('c'):
        print(line.strip())
        continue
    k, d = line.split(' ', 1)
    d = ast.literal_eval(d)
    t = d.get('trace_med', {})
    print(k, d['rc'], d['mismatches'], d['us'], ' '.join(f"{a}={b}" for a, b in t.items()), d.get('trace_max'))
