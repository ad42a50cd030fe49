"""Small workload for compute-sanitizer (tools/sanitize.sh): every kernel family
once on a small scene -- K0/K1/K2 in both MLP modes (tcgen05 + exact), with and
without counters, a sharded render + assemble, the march-segments hook, K3/K4,
and a small bake."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2407_10482_b200 as ng  # noqa: E402

synth = ng.SynthScene(occupancy="bench", occ_base_res=64, L=2, L_C=64, fine_table_len=1 << 12)
dev = ng.Scene(synth)
cams = ng.cameras(3, 48, 40)
for mlp in ("tensor", "exact"):
    ng.render(dev, cams, ng.Opts(mlp=mlp), stats=True)
    ng.render(dev, cams, ng.Opts(mlp=mlp))
sh = torch.stack([ng.render(dev, cams[:1], ng.Opts(shard_world=2, shard_rank=r, shard_tile=16))
                  for r in range(2)])
ng.shard_assemble(sh, 2, 1, 48, 40, 16, 3)
s4 = ng.SynthScene(occupancy="toy", occ_base_res=64, L=4, L_C=32, fine_table_len=1 << 12)
ng.render(ng.Scene(s4), cams[:1], ng.Opts(), stats=True)
words = torch.from_numpy(synth.base_words().view("int64").copy()).cuda()
lv = ng.build_pyramid(words, 64)
ng.build_distance_grid(lv[0], 32)
m = ng.SynthModel(occupancy="bench", occ_base_res=32, L=2, L_C=32, fine_table_len=1 << 12,
                  sigma_lo=-0.5, sigma_hi=-0.5)
ng.bake(m)
torch.cuda.synchronize()
print("sanitize workload done")
