import json, sys, torch
sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parents[2]))
from bench_secondary import f12, c5
dev = torch.device('cuda', 0)
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
r = f12(dev, flush)
print(json.dumps(r, indent=1))
