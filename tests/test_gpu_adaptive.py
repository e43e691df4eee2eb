"""Device adaptive density control (trainer.cpp:167-230)
against the FP64 oracle restatement: same classification (pruned / cloned /
split counts and which kernels), same compaction order, same children
(positions from the same std::mt19937_64 normal draws), Adam state carried for
survivors and zeroed for children; the KATs of test_trainer.cpp:150-231 too."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402


def _engine():
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_2405_20693_b200 as P
    return P, P.Engine()


def _mixed_cloud(m, seed):
    rng = np.random.default_rng(seed)
    s_min = 2e-4
    rho = rng.choice([1e-4, 3e-3, 0.2, 0.8, 2.0], m)
    rho_raw = np.where(rho > 30, rho, np.log(np.expm1(rho))).astype(np.float32)
    pos = rng.uniform(-0.9, 0.9, 3 * m).astype(np.float32)
    scale = rng.choice([0.005, 0.012, 0.03, 0.1], (m, 3)) * rng.uniform(0.8, 1.2, (m, 3))
    scale_raw = np.log(scale - s_min).astype(np.float32).reshape(-1)
    rot = rng.normal(size=(m, 4)).astype(np.float32).reshape(-1)  # unnormalised on purpose
    adam = {k: rng.normal(size=n).astype(np.float32) for k, n in
            zip(O.ADAM_KEYS, (m, m, 3 * m, 3 * m, 3 * m, 3 * m, 4 * m, 4 * m))}
    adam = {k: (np.abs(v) if k.startswith("v_") else v) for k, v in adam.items()}
    count = rng.integers(0, 4, m).astype(np.int32)
    norm = (rng.uniform(0, 2e-4, m) * count).astype(np.float32)
    g3d = rng.normal(size=3 * m).astype(np.float32)
    g3d[:3 * (m // 10)] = 0.0  # zero-norm clones stay in place
    return s_min, rho_raw, pos, scale_raw, rot, adam, count, norm, g3d


@pytest.mark.parametrize("m,seed", [(1, 3), (257, 11), (20000, 29)])
def test_adaptive_control_matches_oracle(m, seed):
    P, eng = _engine()
    s_min, rho_raw, pos, scale_raw, rot, adam, count, norm, g3d = _mixed_cloud(m, seed)
    ext = (2.0, 2.0, 2.0)
    cl = P.GaussianCloud(s_min, rho_raw, pos, scale_raw, rot)
    for k, v in adam.items():
        cl.adam[k].copy_(torch.from_numpy(v))
    cl.grad_count.copy_(torch.from_numpy(count))
    cl.grad2d_norm_accum.copy_(torch.from_numpy(norm))
    cl.grad3d_accum.copy_(torch.from_numpy(g3d))

    oc = O.Cloud(s_min, *(a.astype(np.float64) for a in (rho_raw, pos, scale_raw, rot)))
    st = O.Stats(norm.astype(np.float64), count.copy(), g3d.astype(np.float64))
    oadam = {k: v.astype(np.float64) for k, v in adam.items()}
    onc, oad, ocnt = O.adaptive_control(O.Rng(seed), oc, oadam, st, extent_size=ext)
    draws = O.normal_draws(O.Rng(seed), 6 * ocnt[2])

    nc, cnt = eng.adaptive_control(cl, ext, gauss=torch.from_numpy(draws))
    torch.cuda.synchronize()
    assert cnt == tuple(ocnt)
    assert nc.size() == onc.m
    if m > 100:
        assert min(cnt) > 0, cnt  # the mixture exercises all three actions
    n_kept = onc.m - cnt[1] - 2 * cnt[2]
    got = {k: getattr(nc, k).cpu().numpy().astype(np.float64) for k in ("rho_raw", "pos", "scale_raw", "rot")}
    # survivors are copies (clone parents get act_density_inv(rho/2) rounded to fp32)
    for k in ("pos", "scale_raw", "rot"):
        w = {"pos": 3, "scale_raw": 3, "rot": 4}[k]
        np.testing.assert_array_equal(got[k][: w * n_kept], getattr(onc, k)[: w * n_kept].astype(np.float32))
    np.testing.assert_allclose(got["rho_raw"], onc.rho_raw, rtol=2e-6, atol=1e-6)
    # children: activated values through the inverse activations, fp32 outputs
    np.testing.assert_allclose(got["pos"], onc.pos, rtol=0, atol=2e-6)
    np.testing.assert_allclose(got["scale_raw"], onc.scale_raw, rtol=2e-6, atol=2e-6)
    np.testing.assert_allclose(got["rot"], onc.rot, rtol=0, atol=1e-6)
    for k in O.ADAM_KEYS:
        np.testing.assert_array_equal(nc.adam[k].cpu().numpy(), oad[k].astype(np.float32))
    # statistics reset for the new cloud
    assert not nc.grad_count.any() and not nc.grad2d_norm_accum.any() and not nc.grad3d_accum.any()


def test_adaptive_control_kats():  # test_trainer.cpp:150-212 on the device
    P, eng = _engine()
    # prune only
    cl = P.GaussianCloud(2e-4, np.log(np.expm1([0.3, 1e-4, 0.5])), np.zeros(9), np.log(np.full(9, 0.1 - 2e-4)),
                         np.tile([1.0, 0, 0, 0], 3))
    nc, cnt = eng.adaptive_control(cl, (2, 2, 2))
    assert cnt == (1, 0, 0) and nc.size() == 2
    # clone: small kernel, positional gradient moves the copy
    cl = P.GaussianCloud(2e-4, np.log(np.expm1([0.8])), [0.1, 0.2, 0.3], np.log(np.full(3, 0.01 - 2e-4)),
                         [1.0, 0, 0, 0])
    cl.grad2d_norm_accum.fill_(1.0)
    cl.grad_count.fill_(1)
    cl.grad3d_accum[0] = 1.0
    nc, cnt = eng.adaptive_control(cl, (2, 2, 2))
    assert cnt == (0, 1, 0) and nc.size() == 2
    rho = torch.nn.functional.softplus(nc.rho_raw.double()).cpu().numpy()
    np.testing.assert_allclose(rho, [0.4, 0.4], rtol=1e-6)
    p = nc.pos.view(-1, 3).cpu().numpy()
    assert np.linalg.norm(p[0] - p[1]) > 0
    assert float(nc.adam["m_rho"][1]) == 0.0
    # split: large kernel -> two children with scale / 1.6
    cl = P.GaussianCloud(2e-4, np.log(np.expm1([0.8])), [0.1, 0.2, 0.3], np.log(np.full(3, 0.1 - 2e-4)),
                         [1.0, 0, 0, 0])
    cl.grad2d_norm_accum.fill_(1.0)
    cl.grad_count.fill_(1)
    nc, cnt = eng.adaptive_control(cl, (2, 2, 2), generator=torch.Generator(device="cuda").manual_seed(5))
    assert cnt == (0, 0, 1) and nc.size() == 2
    s = (2e-4 + torch.exp(nc.scale_raw.double())).view(-1, 3).cpu().numpy()
    np.testing.assert_allclose(s[:, 0], [0.1 / 1.6] * 2, rtol=1e-6)
    with pytest.raises(P.ConfigError):
        eng.adaptive_control(cl, (2, 2, 2), split_factor=1.0)
