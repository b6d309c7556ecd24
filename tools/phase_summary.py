"""Sum the TP_PROFILE=1 tuner phase lines of a stderr log: python tools/phase_summary.py log"""
import re
import sys

A = B = H = n = big = 0.0
pat = re.compile(r"candidates (\d+): phase A (\d+) us, phase B (\d+) us \(host enqueue (\d+) us")
for line in open(sys.argv[1]):
    m = pat.search(line)
    if m:
        c, a, b, h = map(int, m.groups())
        n += c; A += a; B += b; H += h
        big += a > 150 * c
print(f"candidates {n:.0f}: phase A {A / 1e3:.0f} ms, phase B {B / 1e3:.0f} ms, host B {H / 1e3:.0f} ms, "
      f"calls with phase A > 150 us/candidate: {big:.0f}")
