"""CPU check of the K7 -> K8 run-partial layout (csrc/partial_layout.cuh):
K8 reads every group of a partial with one 256-bit load, so every partial
must start 32-byte aligned and every group K8 loads must sit in one aligned
4-double group; K7 stages the largest partial in the shared-memory space its
staging tile leaves. Compiled here with g++ (the header is host/device
constexpr), no GPU needed."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SRC = r"""
#define __host__
#define __device__
#include <cstdio>
#include "partial_layout.cuh"
using namespace gmcp_b200;
int main() {
  int bad = 0;
  for (int M = 0; M <= kRunMasters; ++M) {
    const int n = partial_size(M);
    bad += n % 4 != 0;                                    // next partial starts 32-byte aligned
    bad += n < pair_base(M) + M * (M + 1) / 2;            // holds the pair table
    for (int m = 0; m < M; ++m)
      for (int i = 0; i < 3; ++i) bad += (m_base(m) + 4 * i) % 4 != 0;  // a_{m,i} (+ s_m) groups
    bad += pair_base(M) < m_base(M);                      // pair table after the masters
  }
  for (int b = 0; b < 6; ++b) bad += (kSSBase + 12 * b) % 4 != 0;  // SS rows 0-3, 4-7
  bad += kSSBase < 16 || kMBase < kSSBase + 72;           // n | E, g_0..g_2, then 6 SS blocks
  std::printf("%d %d\n", bad, partial_size(kRunMasters));
  return bad != 0;
}
"""


@pytest.mark.skipif(shutil.which("g++") is None, reason="g++ not available")
def test_partial_groups_are_32_byte_aligned(tmp_path):
    src = tmp_path / "layout.cpp"
    src.write_text(SRC)
    exe = tmp_path / "layout"
    subprocess.run(["g++", "-std=c++17", "-I", os.path.join(ROOT, "paper_2605_24339_b200", "csrc"), str(src), "-o",
                    str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    bad, largest = map(int, out.stdout.split())
    assert out.returncode == 0 and bad == 0
    # K7 stages a partial in the 224 doubles its staging tile leaves (assembly.cuh kPst)
    assert largest <= 2 * 16 * 20 - 16 * 17 - 16 * 9
