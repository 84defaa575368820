"""Regenerate tests/golden/bert_base_remat_B4096_120GB.txt: the remat plan
(split list) of the BERT-base seq128 step at B=4096 under a 120 GB budget."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2303_04759_b200.session import ModelConfig, graph_text  # noqa: E402

cfg = ModelConfig.bert_base(B=4096)
cfg.extra["budget"] = 120_000_000_000
with open(os.path.join(ROOT, "tests", "golden", "bert_base_remat_B4096_120GB.txt"), "w") as f:
    f.write(graph_text(cfg, "remat"))
