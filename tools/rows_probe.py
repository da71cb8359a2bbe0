import sys; sys.path.insert(0, ".")
import torch, bench, json
from paper_2405_17381_b200 import ops
dev = torch.device("cuda", 0); s = torch.cuda.current_stream()
print(json.dumps(bench.measure_rows(ops, dev, s, bench.peaks())))
