"""bench.py's config-4 leg (100 random insert/shrink rounds, three release
policies) alone, for A/B of slab policies (GG_PREMAP_CHUNKS=0 / default)."""
import json
import os
import sys
import types
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2209_00103_b200 as gg
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
out = bench.phased_leg(types.SimpleNamespace(quick=False, steps=10, warmup=3), gg, torch, dev)
print(json.dumps({k: out[k] for k in ("ms", "mapped_over_needed_max", "capacity_over_needed_max", "slab")}))
print(json.dumps({p: {k: out[p][k] for k in ("ms", "mapped_over_needed_max", "slab")} for p in ("release_all_policy", "cached_policy")}))
