"""Input generators (no method arithmetic): the FP8 E4M3 quantiser used for the row-f4
storage variant agrees with PyTorch's independent float8_e4m3fn cast."""
import numpy as np
import torch

from paper_2605_18052_b200 import workloads as wl


def test_e4m3_table_and_rounding_match_torch():
    rng = np.random.default_rng(0)
    tab = wl.e4m3_values()
    fin = tab[np.isfinite(tab)]
    x = np.concatenate([rng.normal(0, 3, 100000), rng.normal(0, 0.01, 20000), fin,
                        (fin[:-1] + np.diff(np.sort(fin))[:1].repeat(len(fin) - 1) * 0)]).astype(np.float32)
    x = x[np.abs(x) <= 448]
    code, vals = wl.to_e4m3(x)
    ref = torch.from_numpy(x).to(torch.float8_e4m3fn)
    assert np.array_equal(vals, ref.float().numpy())
    nz = vals != 0  # torch keeps the sign of a zero
    assert np.array_equal(code[nz], ref.view(torch.uint8).numpy()[nz])
    # the code points decode to torch's values; 0x7F / 0xFF are NaN
    allc = torch.arange(256, dtype=torch.uint8).view(torch.float8_e4m3fn).float().numpy()
    assert np.array_equal(np.isnan(tab), np.isnan(allc))
    assert np.array_equal(tab[np.isfinite(tab)], allc[np.isfinite(allc)])
    assert tab[0x7E] == 448.0 and tab[1] == 2.0 ** -9


def test_e4m3_scale_and_saturation():
    code, vals = wl.to_e4m3(np.array([1000.0, -1000.0, 0.75, 3.0], np.float32), scale=0.5)
    assert vals.tolist() == [224.0, -224.0, 0.75, 3.0]
