"""Generate the 2^(k/128) table of csrc/pnms_libm.cuh (exact decimal arithmetic).

Entry k (k = 0..127) is the pair {bits(T_k), bits(H_k) - k * 2^45} with H_k = 2^(k/128)
rounded to the nearest double and T_k = (2^(k/128) - H_k) / H_k rounded to the nearest double,
so that 2^(k/128) ~= H_k * (1 + T_k) — the table layout the table-driven exp of glibc >= 2.28
uses (scale bits are rebuilt as tab[2k+1] + (k_total << 45)).

    python tools/gen_exp_table.py > /tmp/tab.txt
"""
import struct
from decimal import Decimal, getcontext

getcontext().prec = 80


def bits(v: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", v))[0]


def main():
    ln2 = Decimal(2).ln()
    for k in range(128):
        v = (ln2 * k / 128).exp()
        h = float(v)  # correctly rounded
        t = float((v - Decimal(h)) / Decimal(h))
        print(f"    0x{bits(t):016x}ull, 0x{(bits(h) - (k << 45)) & (2**64 - 1):016x}ull,")


if __name__ == "__main__":
    main()
