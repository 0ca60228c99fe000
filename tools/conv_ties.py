"""Near-tie rate of the configs[2] conv encodes (diagnostic)."""
import torch

import paper_2302_03213_b200 as L
from paper_2302_03213_b200 import workloads as W

dev = torch.device("cuda")
for conv, x in W.resnet_convs(dev, batch=16):
    cols = L.im2col(x, 3, 3, 1, 1)
    codes, ties = L.centroid_search_fast(cols, conv.lut.books, return_near_ties=True)
    b = conv.lut.books
    d = torch.cdist(b, b)
    print(conv.in_channels, "rows", cols.shape[0], "ties", ties, "rate", ties / codes.numel(),
          "min centroid sep", float(d[d > 0].min()), "dup centroids", int((d == 0).sum() - d.shape[0] * d.shape[1]))
