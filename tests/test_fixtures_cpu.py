"""Host side of the fixture generator: the detector-noise
entry point sct_add_noise_host consumes the reference's per-view
std::mt19937_64 streams (simulator.cpp:134-158) and must equal the oracle
bit-for-bit after fp32 storage. Pure host code, so it runs without a GPU."""
import numpy as np
import pytest
import torch

from oracle import fixtures as FX
from oracle import oracle as O


def test_add_noise_host_matches_oracle_bitwise():
    from paper_2405_20693_b200 import simulate as S
    clean = np.stack([O.random_image(O.Rng(31 + v), 24, 20, 0.0, 3.0) for v in range(5)]).astype(np.float32)
    noise = S.NoiseParams(i0=1e5, gauss_sigma=10.0, seed=11)
    got = S.add_noise(torch.from_numpy(clean), noise, view0=2).numpy()
    for v in range(5):
        ref = FX.add_noise(clean[v], 1e5, 10.0, 11, 2 + v).astype(np.float32).reshape(20, 24)
        np.testing.assert_array_equal(got[v], ref)
    # no Gaussian term, tiny and huge photon counts (both Poisson regimes of libstdc++)
    for i0 in (7.0, 1e9):
        got = S.add_noise(torch.from_numpy(clean[:2]), S.NoiseParams(i0=i0, gauss_sigma=0.0, seed=5)).numpy()
        for v in range(2):
            ref = FX.add_noise(clean[v], i0, 0.0, 5, v).astype(np.float32).reshape(20, 24)
            np.testing.assert_array_equal(got[v], ref)


def test_add_noise_rejects_bad_photon_count():
    from paper_2405_20693_b200 import ConfigError
    from paper_2405_20693_b200 import simulate as S
    with pytest.raises(ConfigError):
        S.add_noise(torch.zeros(4, 4), S.NoiseParams(i0=0.0))
