"""Merged-FC building blocks on one GPU: the conv part (forward(stop) /
backward(start)) plus the FC head engine (input_grad) reproduce the whole
network's loss and gradient bit for bit -- the identity the merged-FC data
parallel session and asynchronous server rely on."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_1606_04487_b200 import nets  # noqa: E402
from paper_1606_04487_b200.engine import GpuNet  # noqa: E402
from paper_1606_04487_b200.problems import CNNProblem  # noqa: E402


@pytest.mark.parametrize("net,b", [("lenet", 8), ("cifar10_quick", 8), ("caffenet", 4)])
def test_split_at_fc_equals_whole_network(net, b):
    prob = CNNProblem(net, n_examples=16, seed=4, precision="tf32")
    W = torch.from_numpy(prob.initial_weights().astype(np.float32)).cuda()
    idx = torch.arange(b, device="cuda")
    full = prob.engine(b)
    full.gather_batch(prob.data, prob.data_labels, idx)
    loss, G = full.loss_and_grad(W, b)
    loss, G = float(loss.item()), G.clone()

    head_spec, off = nets.fc_head(prob.net)
    conv = GpuNet(prob.net, b, "cuda", "tf32")
    f = conv.first_fc
    head = GpuNet(head_spec, b, "cuda", "tf32", input_grad=True, input_cs=conv.ops[f].inp.cs)
    conv.gather_batch(prob.data, prob.data_labels, idx)
    conv.forward(W, b, stop=f)
    head.input.value[:b].copy_(conv.ops[f].inp.value[:b])
    head.labels[:b].copy_(conv.labels[:b])
    Wfc = W[off:].clone()          # the head stages from an aligned vector
    head.forward(Wfc, b)
    head.backward(b)
    conv.ops[f].inp.grad[:b].copy_(head.input.grad[:b])
    conv.backward(b, start=f)
    torch.cuda.synchronize()
    assert float(head.loss_buf.item()) == loss
    assert torch.equal(conv.grad[:off], G[:off])           # conv gradients
    assert torch.equal(head.grad, G[off:])                 # FC gradients
