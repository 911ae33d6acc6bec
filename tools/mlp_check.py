"""MLP tcgen05 scoring throughput at F=164 (the bench's extra)."""
import sys
sys.path.insert(0, ".")
import json
import torch
import bench

peaks = json.load(open("MEASURED_PEAKS.json")) if __import__("os").path.exists("MEASURED_PEAKS.json") else {}
l2 = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
print(bench.mlp_scoring(l2, torch.cuda.current_stream(), peaks))
