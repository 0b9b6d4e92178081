"""The C ABI's host id map (paper_2502_13965_b200/csrc/idmap.h: active call id -> table row,
open addressing with tombstones) against std::unordered_map under 2M random inserts, overwrites
and erases, with size, lookup and iteration checked every 1000 operations (compiled with g++)."""
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SRC = r"""
#include "idmap.h"
#include <cstdio>
#include <cstdlib>
#include <random>
#include <unordered_map>
int main() {
  IdMap m; std::unordered_map<uint64_t, uint32_t> r; std::mt19937_64 g(1);
  m.reserve(1000);
  std::vector<uint64_t> keys;
  for (int it = 0; it < 2000000; ++it) {
    int op = g() % 3;
    if (op < 2 || keys.empty()) { uint64_t k = g() % 5000 * 0x9E3779B97F4A7C15ull; uint32_t v = g(); m[k] = v; r[k] = v; keys.push_back(k); }
    else { uint64_t k = keys[g() % keys.size()]; m.erase(k); r.erase(k); }
    if (it % 1000 == 0) {
      if (m.size() != r.size()) return 1;
      for (auto& kv : r) { uint32_t* p = m.find(kv.first); if (!p || *p != kv.second) return 2; }
      size_t c = 0; bool bad = false;
      m.for_each([&](uint64_t k, uint32_t& v) { ++c; if (!r.count(k) || r[k] != v) bad = true; });
      if (bad || c != r.size()) return 3;
      if (m.count(~0ull) != r.count(~0ull)) return 4;
    }
  }
  std::printf("ok %zu\n", m.size());
  return 0;
}
"""


def test_idmap_matches_unordered_map(tmp_path):
    c = tmp_path / "t.cpp"
    c.write_text(SRC)
    exe = tmp_path / "t"
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "paper_2502_13965_b200", "csrc"),
                           str(c), "-o", str(exe)])
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0 and out.stdout.startswith("ok"), (out.returncode, out.stdout)
