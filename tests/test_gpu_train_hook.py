"""The training-loop hook (proj/src/train.cpp:26-30,181-199):
projected gradient descent of a softmax classifier with the bi-level
projection applied to the weight on the GPU after every step.  Properties
follow proj/tests/test_train.cpp: feasibility after every step, a huge radius
reproduces unconstrained descent bit for bit, a tight radius drops the
uninformative features while the informative ones keep the accuracy."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def blobs(n, d, informative, classes, sep, seed):
    """Gaussian blobs: class means +/- sep on the informative coordinates."""
    rng = np.random.default_rng(seed)
    inf_idx = rng.choice(d, informative, replace=False)
    signs = np.zeros((classes, d))
    signs[:, inf_idx] = rng.choice([-1.0, 1.0], size=(classes, informative))
    if classes == 2:
        signs[0, inf_idx], signs[1, inf_idx] = -1.0, 1.0
    labels = rng.integers(0, classes, n)
    x = sep * signs[labels] + rng.normal(size=(n, d))
    return x.astype(np.float32), labels, inf_idx


def train(x, labels, classes, eta, steps, lr, q="inf", feature_dim=1, graph=False):
    import torch
    import paper_2405_02086_b200.hooks as hooks
    dev = torch.device("cuda")
    xt = torch.from_numpy(x).to(dev)
    yt = torch.from_numpy(labels).to(dev)
    g = torch.Generator(device="cpu").manual_seed(3)
    w0 = (0.01 * torch.randn(classes, x.shape[1], generator=g)).to(dev)
    w = torch.nn.Parameter(w0 if feature_dim == 1 else w0.t().contiguous())
    b = torch.nn.Parameter(torch.zeros(classes, device=dev))
    hook = hooks.FeatureProjector(w, eta, q=q, feature_dim=feature_dim) if eta is not None else None
    if hook:
        hook()

    def step():
        logits = xt @ (w.t() if feature_dim == 1 else w) + b
        loss = torch.nn.functional.cross_entropy(logits, yt)
        gw, gb = torch.autograd.grad(loss, (w, b))
        with torch.no_grad():
            w.sub_(lr * gw)
            b.sub_(lr * gb)
        if hook:
            hook()
        return loss

    history = []
    for _ in range(steps):
        step()
        wk = (w.detach() if feature_dim == 1 else w.detach().t()).double().cpu().numpy()
        history.append(wk)
    with torch.no_grad():
        acc = float(((xt @ (w.t() if feature_dim == 1 else w) + b).argmax(1) == yt).float().mean())
    return history, acc, hook


def group_norm(wk, q):
    # features are the columns of the (classes x features) weight
    return O.matrix_pq_norm(wk, "1", q)


@pytest.mark.parametrize("q", ["inf", "2"])
def test_projected_descent_feasible_and_sparse(q):
    x, labels, inf_idx = blobs(600, 50, 5, 3, 2.5, seed=7)
    eta = 1.5
    hist, acc, hook = train(x, labels, 3, eta, 60, 0.5, q=q)
    for wk in hist:
        assert group_norm(wk, q) <= eta * (1 + 1e-6)
    last = hist[-1]
    zero = np.all(last == 0.0, axis=0)
    survivors = set(np.flatnonzero(~zero))
    assert survivors and survivors <= set(inf_idx), survivors  # only informative features survive
    assert acc > 0.9, acc
    assert hook.zero_features() == int(zero.sum())


def test_huge_radius_reproduces_unconstrained_descent():  # test_train.cpp:70-78
    x, labels, _ = blobs(200, 12, 4, 2, 2.0, seed=17)
    a, _, _ = train(x, labels, 2, 1e12, 25, 0.1)
    b, _, _ = train(x, labels, 2, None, 25, 0.1)
    assert all(np.array_equal(u, v) for u, v in zip(a, b))


def test_rows_layout_matches_columns_layout():
    """feature_dim=0 (the reference's W, features x classes, projected through a
    transpose) gives the same weights as the in-place column layout."""
    x, labels, _ = blobs(300, 20, 4, 3, 2.0, seed=5)
    a, _, _ = train(x, labels, 3, 1.0, 20, 0.3, feature_dim=1)
    b, _, _ = train(x, labels, 3, 1.0, 20, 0.3, feature_dim=0)
    for u, v in zip(a, b):
        np.testing.assert_allclose(u, v, rtol=1e-5, atol=1e-7)


def test_hook_inside_a_captured_training_step():
    import torch
    import paper_2405_02086_b200.hooks as hooks
    dev = torch.device("cuda")
    x, labels, _ = blobs(256, 32, 4, 2, 2.0, seed=9)
    xt, yt = torch.from_numpy(x).to(dev), torch.from_numpy(labels).to(dev)
    w = torch.zeros(2, 32, device=dev)
    w.normal_(generator=torch.Generator(device=dev).manual_seed(1)).mul_(0.01)
    w_eager = w.clone()
    hook = hooks.FeatureProjector(w, 0.8)
    hook_e = hooks.FeatureProjector(w_eager, 0.8)

    def step(wt, hk):
        p = torch.softmax(xt @ wt.t(), dim=1)
        p[torch.arange(len(yt), device=dev), yt] -= 1.0
        wt.sub_(0.2 * (p.t() @ xt) / len(yt))
        hk()

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step(w, hook)  # warm-up outside capture
        step(w_eager, hook_e)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            step(w, hook)
        for _ in range(10):
            g.replay()
            step(w_eager, hook_e)
    torch.cuda.synchronize()
    assert torch.equal(w, w_eager)
    assert O.matrix_pq_norm(w.double().cpu().numpy(), "1", "inf") <= 0.8 * (1 + 1e-6)
