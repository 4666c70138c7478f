"""GPU distillation: the oracle restatement of one training
step against the reference's own outputs (CPU), and the CUDA trainer against
both (GPU).  Fixture: tests/golden/train_step.npz (make_golden.py gen_train)."""

import numpy as np
import pytest

from oracle import nedf_oracle as O


def _oracle_model(z):
    return O.parse_nedm(z["raw"].tobytes())


def _blocks(flat, model):
    out, k = [], 0
    for w, b in model.weights:
        for a in (w, b):
            out.append(flat[k:k + a.size].reshape(a.shape))
            k += a.size
    return out


def test_oracle_training_step_matches_reference(golden):
    z = golden("train_step.npz")
    m = _oracle_model(z)
    hit = z["hit"].astype(bool)
    total, parts, grads = O.loss_and_grads(m, z["feats"], z["coarse"], z["fine"], hit)
    assert total == pytest.approx(float(z["total"]), rel=1e-12)
    np.testing.assert_allclose(parts, z["parts"], rtol=1e-12)
    g = np.concatenate([x.ravel() for x in grads])
    np.testing.assert_allclose(g, z["grads"], rtol=1e-9, atol=1e-15)
    params = [a.copy() for a in O.flat_params(m)]
    O.adam_step(params, grads, [np.zeros_like(p) for p in params], [np.zeros_like(p) for p in params], 1)
    np.testing.assert_allclose(np.concatenate([p.ravel() for p in params]), z["params_after"], rtol=0, atol=1e-15)


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


@pytest.mark.gpu
def test_gpu_loss_gradients_and_adam(golden):
    from paper_2308_04669_b200 import model, train
    z = golden("train_step.npz")
    m = model.loads_nedf(z["raw"].tobytes())
    tr = train.Trainer(m, max_batch=256)
    hit = z["hit"].astype(bool)
    tr.set_batch(z["feats"], np.where(hit, z["coarse"], -1), np.where(hit, z["fine"], -1), hit)
    total, parts = tr.loss_and_grads()
    assert total == pytest.approx(float(z["total"]), rel=2e-5)
    np.testing.assert_allclose(parts, z["parts"], rtol=2e-5)
    g = tr.grads().astype(np.float64)
    om = _oracle_model(z)
    for got, ref in zip(_blocks(g, om), _blocks(z["grads"], om)):   # every parameter block, fp32 vs fp64
        assert _rel(got, ref) < 2e-4
    tr.adam_step()
    p = tr.params().astype(np.float64)
    ref = z["params_after"]
    close = np.abs(p - ref) <= 1e-6 + 1e-6 * np.abs(ref)
    # the first Adam step moves each weight by ~lr * sign(g); gradients within fp32 noise of
    # zero may take the other sign
    assert close.mean() > 0.999
    assert np.abs(p - ref).max() <= 2 * 5e-4 + 1e-6


@pytest.mark.gpu
def test_gpu_batch_targets_match_reference(golden):
    """RaySampler(seed 7) + GPU encoding, sphere tracing and bin quantisation give the
    reference's batch (model.py:210-235)."""
    from paper_2308_04669_b200 import fields, geometry, model, train
    z = golden("train_step.npz")
    m = model.loads_nedf(z["raw"].tobytes())
    oracle = fields.AnalyticOracle(fields.Sphere(geometry.vec3(0, 0, 0), 1.0))
    tr = train.Trainer(m, max_batch=256)
    b = train.build_training_batch(oracle, train.RaySampler(m.relaxed_box), tr, np.random.default_rng(7), 256)
    assert b.n == len(z["hit"])
    total, parts = tr.loss_and_grads()
    assert total == pytest.approx(float(z["total"]), rel=2e-5)
    np.testing.assert_allclose(parts, z["parts"], rtol=2e-5)


@pytest.mark.gpu
def test_gpu_training_reduces_loss_and_updates_model():
    from paper_2308_04669_b200 import fields, geometry, model, train
    oracle = fields.AnalyticOracle(fields.Sphere(geometry.vec3(0, 0, 0), 1.0))
    m = model.new_model(oracle, np.random.default_rng(0), model.PROFILES["desk"])
    before = m.nedm_bytes()
    losses = train.train(m, oracle, np.random.default_rng(1), iterations=60, batch_size=512, lr=1e-3)
    assert len(losses) == 60 and np.all(np.isfinite(losses))
    assert np.mean(losses[-10:]) < 0.8 * np.mean(losses[:5])
    assert m.nedm_bytes() != before
    o, d = train.RaySampler(m.relaxed_box).sample(np.random.default_rng(2), 64)
    mu, alpha = model.query_rays(m, o, d)        # the trained weights are live
    assert mu.shape == (64,)
