"""Config 5's training harness: the Llama-style model's parameter list is the 953M optimizer workload, and a
small model trains through the DASH step on the GPU."""
import pytest
import torch

from paper_2602_02016_b200.llama import LlamaShape
from tests.golden.cases import llama_953m


def test_param_shapes_are_the_953m_workload():
    shape = LlamaShape()
    assert shape.param_shapes() == llama_953m()
    assert sum(int(torch.Size(s).numel()) for s in shape.param_shapes()) == 953_223_168


@pytest.mark.gpu
def test_small_llama_trains_with_dash():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2602_02016_b200.llama import TrainStep
    from paper_2602_02016_b200.shampoo import LrSchedule, ShampooConfig, SolverConfig

    shape = LlamaShape(dim=128, layers=2, ffn=256, vocab=512, heads=4)
    cfg = ShampooConfig(block_size=64, lr=LrSchedule(base=3e-3),
                        solver=SolverConfig(method="ndb", tolerance=0.0, max_iters=10))
    trainer = TrainStep(shape, cfg, "cuda", seed=0)
    g = torch.Generator(device="cuda").manual_seed(1)
    tokens = torch.randint(0, shape.vocab, (4, 65), device="cuda", generator=g)
    losses = [float(trainer(tokens)) for _ in range(8)]
    assert all(torch.isfinite(torch.tensor(losses)))
    assert losses[-1] < losses[0] - 0.1, losses
