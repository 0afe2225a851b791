import numpy as np, sys
sys.path.insert(0, '.')
import paper_2201_05500_b200 as kp
from paper_2201_05500_b200.data import make_batch
tr = kp.Trainer(table_capacity=8, n_workers=1, embedding_dim=4, hidden=[])
bt = make_batch(64, V=10**6, zipf_s=None, nnz=4, seed=0)
try:
    tr.train_batch(bt.offs, bt.keys, bt.labels)
except Exception as e:
    print(type(e).__name__, e)
