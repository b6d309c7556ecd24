"""Measure per-layer latency vs a trivial kernel floor (debug)."""
import sys; sys.path.insert(0,'.')
import torch, json
from paper_2008_03602_b200 import datagen, tp, workloads as wl
tp.init(0)
