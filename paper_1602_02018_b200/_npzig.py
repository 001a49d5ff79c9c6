"""numpy's standard-normal generator, restated for a bit-exact device port.

Parity requires the reference's seeded numpy draws (spectrum.py:84,
features.py:63).  numpy's ``Generator(PCG64).standard_normal`` is:

* PCG64: 128-bit LCG, ``state = state * M + inc`` then output
  ``rotr64(hi ^ lo, hi >> 58)`` (XSL-RR), one uint64 per step;
* the 256-layer ziggurat of ``random_standard_normal``: a uint64 gives the
  layer (low 8 bits), a sign bit and a 52-bit magnitude; 99.3 % of draws return
  ``magnitude * wi[layer]`` at once, the rest take the wedge / tail tests that
  consume extra doubles (``(u >> 11) * 2**-53``).

The ziggurat tables are read from numpy's own compiled module at run time (they
are data of the installed numpy, not of the reference package) and checked
against numpy's output before use.  ``NormalStream`` below is the pure-Python
statement of the algorithm used to validate the tables and the device port.
"""

from __future__ import annotations

import glob
import math
import os
import struct
from functools import lru_cache

import numpy as np

PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645
MASK128 = (1 << 128) - 1
MASK64 = (1 << 64) - 1
ZIG_R = 3.6541528853610087963519472518  # tail start of the 256-layer normal ziggurat
ZIG_INV_R = 0.27366123732975827203338247596
ZIG_EXP_R = 7.69711747013104972  # tail start of the 256-layer exponential ziggurat


def _elf_symbols(path: str, names: set[str]) -> dict[str, bytes]:
    """Bytes of named data symbols of an ELF64 shared object (via .symtab/.dynsym)."""
    with open(path, "rb") as fh:
        data = fh.read()
    if data[:4] != b"\x7fELF" or data[4] != 2:
        raise ValueError("not an ELF64 file")
    shoff, = struct.unpack_from("<Q", data, 0x28)
    shentsize, shnum, _ = struct.unpack_from("<HHH", data, 0x3A)
    sections = [struct.unpack_from("<IIQQQQIIQQ", data, shoff + i * shentsize) for i in range(shnum)]
    out: dict[str, bytes] = {}
    for sec in sections:
        _, sh_type, _, _, sh_offset, sh_size, sh_link, _, _, sh_entsize = sec
        if sh_type not in (2, 11) or not sh_entsize:  # SHT_SYMTAB, SHT_DYNSYM
            continue
        strtab = sections[sh_link]
        for k in range(sh_size // sh_entsize):
            st_name, _, _, st_shndx, st_value, st_size = struct.unpack_from("<IBBHQQ", data, sh_offset + k * sh_entsize)
            if st_shndx == 0 or st_shndx >= len(sections):
                continue
            name_off = strtab[4] + st_name
            name = data[name_off : data.index(b"\x00", name_off)].decode("ascii", "replace")
            if name in names and name not in out:
                tsec = sections[st_shndx]
                foff = tsec[4] + (st_value - tsec[3])
                out[name] = data[foff : foff + st_size]
    return out


def _find_tables(names: tuple[str, str, str]):
    base = os.path.dirname(np.random.__file__)
    for path in sorted(glob.glob(os.path.join(base, "_generator*.so"))) + sorted(glob.glob(os.path.join(base, "*.so"))):
        try:
            syms = _elf_symbols(path, set(names))
        except (OSError, ValueError, struct.error):
            continue
        if len(syms) == 3 and all(len(v) == 2048 for v in syms.values()):
            k, w, f = (syms[n] for n in names)
            return (np.frombuffer(k, dtype="<u8").copy(), np.frombuffer(w, dtype="<f8").copy(),
                    np.frombuffer(f, dtype="<f8").copy())
    return None


@lru_cache(maxsize=1)
def exponential_tables() -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(ke uint64[256], we float64[256], fe float64[256]) of the installed numpy, verified."""
    tabs = _find_tables(("ke_double", "we_double", "fe_double"))
    if tabs is None:
        raise RuntimeError("numpy's exponential ziggurat tables were not found")
    verify_exponential_tables(*tabs)
    return tabs


@lru_cache(maxsize=1)
def ziggurat_tables() -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """(ki uint64[256], wi float64[256], fi float64[256]) of the installed numpy."""
    base = os.path.dirname(np.random.__file__)
    for path in sorted(glob.glob(os.path.join(base, "_generator*.so"))) + sorted(glob.glob(os.path.join(base, "*.so"))):
        try:
            syms = _elf_symbols(path, {"ki_double", "wi_double", "fi_double"})
        except (OSError, ValueError, struct.error):
            continue
        if len(syms) == 3 and all(len(v) == 2048 for v in syms.values()):
            ki = np.frombuffer(syms["ki_double"], dtype="<u8").copy()
            wi = np.frombuffer(syms["wi_double"], dtype="<f8").copy()
            fi = np.frombuffer(syms["fi_double"], dtype="<f8").copy()
            verify_tables(ki, wi, fi)
            return ki, wi, fi
    raise RuntimeError("numpy's ziggurat tables were not found; device parity RNG unavailable")


class NormalStream:
    """numpy's Generator(PCG64).standard_normal, one draw at a time (pure Python).

    ``exp_tables`` enables ``exponential()`` / ``geometric()`` as well."""

    def __init__(self, state: int, inc: int, tables, exp_tables=None):
        self.s, self.inc = state, inc
        self.ki, self.wi, self.fi = tables
        self.ke, self.we, self.fe = exp_tables if exp_tables is not None else (None, None, None)
        self.raw_count = 0

    def next_u64(self) -> int:
        self.s = (self.s * PCG_MULT + self.inc) & MASK128
        self.raw_count += 1
        hi, lo = self.s >> 64, self.s & MASK64
        x, r = hi ^ lo, hi >> 58
        return ((x >> r) | (x << ((64 - r) & 63))) & MASK64

    def next_double(self) -> float:
        return (self.next_u64() >> 11) * (1.0 / 9007199254740992.0)

    def normal(self) -> float:
        while True:
            r = self.next_u64()
            idx = r & 0xFF
            r >>= 8
            rabs = (r >> 1) & 0x000FFFFFFFFFFFFF
            x = rabs * float(self.wi[idx])
            if r & 1:
                x = -x
            if rabs < int(self.ki[idx]):
                return x
            if idx == 0:
                while True:
                    xx = -ZIG_INV_R * math.log1p(-self.next_double())
                    yy = -math.log1p(-self.next_double())
                    if yy + yy > xx * xx:
                        return -(ZIG_R + xx) if (rabs >> 8) & 1 else ZIG_R + xx
            elif (float(self.fi[idx - 1]) - float(self.fi[idx])) * self.next_double() + float(self.fi[idx]) < math.exp(
                -0.5 * x * x
            ):
                return x


    def exponential(self) -> float:
        """numpy's random_standard_exponential (exponential ziggurat)."""
        while True:
            ri = self.next_u64() >> 3
            idx = ri & 0xFF
            ri >>= 8
            x = ri * float(self.we[idx])
            if ri < int(self.ke[idx]):
                return x
            if idx == 0:
                return ZIG_EXP_R - math.log1p(-self.next_double())
            if (float(self.fe[idx - 1]) - float(self.fe[idx])) * self.next_double() + float(self.fe[idx]) < math.exp(-x):
                return x

    def geometric(self, p: float) -> int:
        """numpy's random_geometric: search for p >= 1/3, inversion otherwise."""
        if p >= 0.333333333333333333333333:
            x, total, prod, q = 1, p, p, 1.0 - p
            u = self.next_double()
            while u > total:
                prod *= q
                total += prod
                x += 1
            return x
        z = math.ceil(-self.exponential() / math.log1p(-p))
        return (1 << 63) - 1 if z >= 9.223372036854776e18 else int(z)


def pcg_state(rng: np.random.Generator) -> tuple[int, int]:
    """128-bit state and increment of a PCG64 generator.  A buffered 32-bit half
    (``has_uint32``) is not part of the 64-bit stream the double draws consume; callers that
    advance the generator carry it over (``_signals.device_normal_block``)."""
    st = rng.bit_generator.state
    if st["bit_generator"] != "PCG64":
        raise ValueError("parity RNG needs a PCG64 generator")
    return int(st["state"]["state"]), int(st["state"]["inc"])


def verify_tables(ki, wi, fi, draws: int = 20000) -> None:
    """The restated generator must reproduce numpy draw for draw (incl. slow paths)."""
    for seed in (0, 12345):
        rng = np.random.default_rng(seed)
        s, inc = pcg_state(rng)
        ref = rng.standard_normal(draws)
        ns = NormalStream(s, inc, (ki, wi, fi))
        got = np.array([ns.normal() for _ in range(draws)])
        if not np.array_equal(got, ref):
            raise RuntimeError("ziggurat tables do not reproduce numpy's standard_normal")
        if (ns.s, ns.inc) != pcg_state(rng):
            raise RuntimeError("PCG64 stream position diverged from numpy")


def verify_exponential_tables(ke, we, fe, draws: int = 20000) -> None:
    """The restated exponential / geometric draws must reproduce numpy's."""
    for seed in (0, 12345):
        rng = np.random.default_rng(seed)
        s, inc = pcg_state(rng)
        ref = rng.standard_exponential(draws)
        ns = NormalStream(s, inc, (None, None, None), (ke, we, fe))
        got = np.array([ns.exponential() for _ in range(draws)])
        if not np.array_equal(got, ref) or (ns.s, ns.inc) != pcg_state(rng):
            raise RuntimeError("exponential tables do not reproduce numpy's standard_exponential")
