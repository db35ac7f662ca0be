import sys, os, json, numpy as np, torch
sys.path.insert(0, '/root/repo')
import bench
print(json.dumps(bench.c1_measure(0)))
