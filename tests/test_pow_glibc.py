"""csrc/pow_glibc.cuh (glibc's pow restated for the device) built for the host
and compared bit for bit with the host's libm pow() -- the function CPython's
`**` calls -- on the bases the IDM produces (speed ratios, gap ratios) and on
extreme ranges (subnormal and huge results)."""

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = r'''
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include "pow_glibc.cuh"
double (*volatile libm_pow)(double, double) = std::pow;
int main(int argc, char** argv) {
  long n = atol(argv[1]);
  std::mt19937_64 rng(atol(argv[2]));
  long bad = 0;
  const double ys[] = {4.0, 2.0, 3.0, 0.5, 1.5, 4.25};
  for (long k = 0; k < n; k++) {
    const double y = ys[k % 6];
    double x;
    const uint64_t u = rng();
    switch ((k / 6) % 5) {
      case 0: x = std::ldexp((double)(u >> 11), -53) * 1.3; break;   // v / v0_eff
      case 1: x = std::ldexp((double)(u >> 11), -53) * 2e6; break;   // s* / gap
      case 2: x = std::ldexp(1.0 + std::ldexp((double)(u >> 12), -52), (int)(rng() % 200) - 100); break;
      case 3: x = std::ldexp(1.0 + std::ldexp((double)(u >> 12), -52), (int)(rng() % 40) - 275); break;
      default: x = std::ldexp(1.0 + std::ldexp((double)(u >> 12), -52), (int)(rng() % 30) + 230); break;
    }
    const double a = tsb::glibc_pow::pow(x, y), b = libm_pow(x, y);
    if (std::memcmp(&a, &b, 8) != 0) {
      if (bad < 3) printf("x=%a y=%a mine=%a libm=%a\n", x, y, a, b);
      bad++;
    }
  }
  printf("POW_CHECK %ld %ld\n", n, bad);
  return 0;
}
'''


def test_device_pow_is_bit_exact_with_libm(tmp_path):
    src = tmp_path / "powcheck.cpp"
    exe = tmp_path / "powcheck"
    src.write_text(SRC)
    subprocess.run(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-builtin",
                    "-I", os.path.join(ROOT, "paper_2405_12520_b200", "csrc"), str(src), "-o", str(exe), "-lm"],
                   check=True)
    out = subprocess.run([str(exe), "6000000", "3"], capture_output=True, text=True, check=True).stdout
    line = [x for x in out.splitlines() if x.startswith("POW_CHECK")][0]
    assert line.split()[2] == "0", out
