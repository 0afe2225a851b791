"""Timing experiments on the first layer's forward (KP_H3_DBG modes): one
configs[1] training step, errors from garbage modes ignored. Run under ncu."""
import sys
sys.path.insert(0, 'tests')
from helpers import trainer_kwargs
from oracle import oracle as O
import paper_2201_05500_b200 as kp
from paper_2201_05500_b200.data import make_batch
B = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
cfg = O.TrainerCfg(n_workers=1, k=1, minibatch_size=B, embedding_dim=64, n_slots=100,
                   hidden=(256, 128), pooling="sum", activation="relu", alpha=0.01, sparse_lr=0.05)
tr = kp.Trainer(table_capacity=1 << 27, **trainer_kwargs(vars(cfg)))
bt = make_batch(B, V=10**8, zipf_s=1.1, n_slots=100, seed=1)
for i in range(2):
    try:
        tr.train_batch(bt.offs, bt.keys, bt.labels, slots=bt.slots)
    except Exception as e:  # noqa: BLE001 (garbage timing modes trip the finite checks)
        print("step", i, type(e).__name__)
