"""Checkpoint / resume: host-only round trip and
architecture checks of paper_1302_1690_b200.checkpoint, and (marked gpu) a resumed training
step through MPFNet.save / load."""
import numpy as np
import pytest

import mpf_synth as S
from paper_1302_1690_b200.checkpoint import load_checkpoint, save_checkpoint


def test_round_trip_and_architecture_checks(tmp_path):
    cfg = S.CONFIGS["cfg2"]
    params = S.init_params(cfg).astype(np.float32)
    path = str(tmp_path / "ck.npz")
    save_checkpoint(path, cfg.layers, cfg.P, 1, params, step=17)
    ck = load_checkpoint(path, cfg.layers, cfg.P, 1, params.size)
    assert ck["step"] == 17 and ck["patch"] == cfg.P and ck["in_channels"] == 1
    assert ck["params"].dtype == np.float32 and np.array_equal(ck["params"], params)
    other = S.CONFIGS["cfg5"]
    with pytest.raises(ValueError, match="layer list"):
        load_checkpoint(path, other.layers)
    with pytest.raises(ValueError, match="patch"):
        load_checkpoint(path, cfg.layers, cfg.P + 1)
    with pytest.raises(ValueError, match="in_channels"):
        load_checkpoint(path, cfg.layers, cfg.P, 4)
    with pytest.raises(ValueError, match="parameters"):
        load_checkpoint(path, cfg.layers, cfg.P, 1, params.size + 1)


def test_rejects_foreign_files(tmp_path):
    path = str(tmp_path / "x.npz")
    np.savez(path, format=np.array("something-else"), version=np.int32(1))
    with pytest.raises(ValueError, match="not an"):
        load_checkpoint(path)


@pytest.mark.gpu
def test_net_save_load_resumes_bitwise(tmp_path):
    """A step from a loaded checkpoint equals the step from the saved state, bitwise."""
    import torch
    from paper_1302_1690_b200.net import MPFNet
    cfg = S.CONFIGS["cfg2"]
    images, labels = S.make_batch(cfg, [0, 1])
    img, lab = torch.tensor(images, device="cuda"), torch.tensor(labels, device="cuda")
    a = MPFNet(cfg.layers, cfg.P, cfg.H, cfg.W, max_images=2)
    a.set_params(S.init_params(cfg).astype(np.float32))
    a.train_step(img, lab)
    a.sgd_step(cfg.lr, 0.5)
    path = str(tmp_path / "ck.npz")
    a.save(path, step=1)
    b = MPFNet(cfg.layers, cfg.P, cfg.H, cfg.W, max_images=2)
    assert b.load(path) == 1
    la, lb = a.train_step(img, lab), b.train_step(img, lab)
    torch.cuda.synchronize()
    assert torch.equal(la, lb) and torch.equal(a.grads, b.grads)
