import os, sys, numpy as np
sys.path.insert(0, 'tests')
from helpers import trainer_kwargs
from oracle import oracle as O
import paper_2201_05500_b200 as kp
from paper_2201_05500_b200.data import make_batch
B, S, e = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
cfg = O.TrainerCfg(n_workers=1, k=2, minibatch_size=B, embedding_dim=e, n_slots=S,
                   hidden=(256, 128), pooling="sum", activation="relu", alpha=0.02, sparse_lr=0.1)
tr = kp.Trainer(table_capacity=1 << 20, **trainer_kwargs(vars(cfg)))
bt = make_batch(B, V=10**6, zipf_s=1.1, n_slots=S, seed=300)
r = tr.train_batch(bt.offs, bt.keys, bt.labels, slots=bt.slots, predict_first=False)
print("loss", r["loss"])
