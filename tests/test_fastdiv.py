"""Host check of the render kernels' division by launch-invariant divisors
(paper_2402_03106_b200/csrc/fastdiv.h): the header is compiled here with g++
and its quotient/remainder compared with the integer division of C for edge
divisors (1, powers of two and their neighbours, 2^32 - 1, the workloads'
pixel / bin / sample counts) against edge and random numerators."""
from __future__ import annotations

import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SRC = r"""
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "fastdiv.h"
static uint64_t st = 88172645463325252ull;
static uint32_t rnd() { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return (uint32_t)st; }
int main() {
  std::vector<uint32_t> ds = {1, 2, 3, 5, 7, 10, 16, 100, 120, 128, 255, 256, 257, 1000, 1023, 1024, 1025, 4096,
                              16384, 65535, 65536, 65537, 1048576, 1000000, 2147483647u, 2147483648u,
                              2147483649u, 4294967295u, 4294967294u};
  for (int i = 0; i < 200; ++i) ds.push_back(rnd() | 1u);
  for (int i = 0; i < 200; ++i) ds.push_back(1u + rnd() % 5000u);
  long bad = 0, n_checked = 0;
  for (uint32_t d : ds) {
    const FastDiv f = fastdiv_make(d);
    std::vector<uint32_t> ns = {0, 1, 2, d - 1, d, d + 1, 2 * d - 1, 2 * d, 4294967295u, 4294967294u,
                                2147483647u, 2147483648u};
    const uint64_t top = 4294967295ull / d * d;
    ns.push_back((uint32_t)top);
    ns.push_back((uint32_t)(top - 1));
    for (int i = 0; i < 20000; ++i) ns.push_back(rnd());
    for (int i = 0; i < 2000; ++i) ns.push_back(rnd() % 100000u);
    for (uint32_t n : ns) {
      uint32_t r;
      const uint32_t q = fastdiv_divmod(n, f, r);
      ++n_checked;
      if (q != n / d || r != n % d) {
        if (bad < 5) std::printf("BAD n=%u d=%u q=%u r=%u\n", n, d, q, r);
        ++bad;
      }
    }
  }
  std::printf("checked %ld bad %ld\n", n_checked, bad);
  return bad != 0;
}
"""


def test_fastdiv_matches_integer_division(tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text(_SRC)
    exe = tmp_path / "t"
    inc = os.path.join(ROOT, "paper_2402_03106_b200", "csrc")
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", inc, str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "bad 0" in out.stdout
