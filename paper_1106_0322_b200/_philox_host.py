"""Host-side Philox4x64-10 for the few scalars the host needs.

The resampling uniform u = _stream(seed, 2, t).random() / N (reference
smc.py:289, 421) is a single draw; computing it on the host avoids a device
round trip.  Same bijection and counter convention as csrc/philox.cuh.
"""

_M0, _M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
_W0, _W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B
_MASK = (1 << 64) - 1


def philox_block(k0: int, k1: int, index: int):
    """Block `index` of stream key (k0, k1): counter index + 1."""
    c = [(index + 1) & _MASK, (index + 1) >> 64, 0, 0]
    for _ in range(10):
        p0 = _M0 * c[0]
        p1 = _M1 * c[2]
        c = [((p1 >> 64) ^ c[1] ^ k0) & _MASK, p1 & _MASK, ((p0 >> 64) ^ c[3] ^ k1) & _MASK, p0 & _MASK]
        k0 = (k0 + _W0) & _MASK
        k1 = (k1 + _W1) & _MASK
    return c


def stream_key(seed: int, tag: int, t: int = 0, i: int = 0):
    return int(seed) & _MASK, ((int(tag) << 58) | (int(t) << 34) | int(i)) & _MASK


def first_uniform(seed: int, tag: int, t: int = 0, i: int = 0) -> float:
    k0, k1 = stream_key(seed, tag, t, i)
    return (philox_block(k0, k1, 0)[0] >> 11) * 2.0**-53
