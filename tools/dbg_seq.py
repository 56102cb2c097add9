import os, sys, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, json
import bench
which = sys.argv[1:]
for w in which:
    gc.collect(); torch.cuda.empty_cache()
    try:
        r = getattr(bench, w)()
        print(w, "OK", r["ms"])
    except AssertionError as e:
        print(w, "ASSERT", e)
