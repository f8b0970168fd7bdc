"""The weight-plane word encoding (paper_0911_2900_b200/csrc/plane.cu) restated in numpy: a
candidate's weight relative to the agent is one integer add on its plane word, read as fp32 with
the sign dropped -- exactly m_c * 2^(C_p - C_c) for every |C_p - C_c| <= 60, across the
mod-256 wrap of the stored exponent (CPU; no device)."""
import numpy as np


def word(C, mant):  # bits 30..23 = (-C) mod 256, bits 22..0 = mantissa
    return ((((-C) & 0xFF).astype(np.uint32) << np.uint32(23)) | mant.astype(np.uint32)).astype(np.uint32)


def offset(own):  # A_p = ((C_p + 127) mod 256) << 23 from the agent's own word
    return (((np.uint32(127) - (own >> np.uint32(23))) & np.uint32(255)) << np.uint32(23)).astype(np.uint32)


def test_one_add_weight_is_exact():
    r = np.random.default_rng(11)
    n = 200000
    Cp = r.integers(-100000, 100000, n)
    d = r.integers(-60, 61, n)
    Cc = Cp - d
    mant = r.integers(0, 1 << 23, n)
    own = word(Cp, r.integers(0, 1 << 23, n))  # an unflagged centre
    w = word(Cc, mant) | (r.integers(0, 2, n).astype(np.uint32) << np.uint32(31))  # flag bits of candidates are ignored
    got = np.abs((w + offset(own)).astype(np.uint32).view(np.float32)).astype(np.float64)
    want = (1.0 + mant / 2.0**23) * np.exp2(d.astype(np.float64))
    assert (got == want).all()


def test_wrap_of_the_stored_exponent():
    # balls straddling a multiple of 256 in C: the add wraps mod 256 and still lands on the weight
    Cp = np.array([255, 256, 0, -1, 511, 512, 1023], np.int64)
    for dd in (-60, -1, 0, 1, 60):
        Cc = Cp - dd
        mant = np.full(len(Cp), 12345)
        got = np.abs((word(Cc, mant) + offset(word(Cp, mant))).astype(np.uint32).view(np.float32))
        assert (got.astype(np.float64) == (1.0 + 12345 / 2.0**23) * 2.0**dd).all()
