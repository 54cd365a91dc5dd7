// stdsort_probe.cpp -- TEST INFRASTRUCTURE ONLY.
// Calls this toolchain's libstdc++ std::sort exactly the way scipy's
// csr_sort_indices does (std::vector<std::pair<I,T>>, comparator on .first
// only) so tests/test_oracle.py can check the introsort restatement in
// gift_oracle.c (and, on the GPU, csrc/introsort.cuh) permutation for
// permutation, including the heapsort fallback on adversarial inputs.
#include <algorithm>
#include <cstdint>
#include <utility>
#include <vector>

static bool kv_pair_less(const std::pair<int64_t, double>& x, const std::pair<int64_t, double>& y) {
  return x.first < y.first;
}

extern "C" void probe_std_sort_perm(int64_t n, const int64_t* keys, int64_t* perm_out) {
  std::vector<std::pair<int64_t, double>> tmp(n);
  for (int64_t i = 0; i < n; ++i) tmp[i] = std::make_pair(keys[i], (double)i);
  std::sort(tmp.begin(), tmp.end(), kv_pair_less);
  for (int64_t i = 0; i < n; ++i) perm_out[i] = (int64_t)tmp[i].second;
}

// McIlroy's "killer adversary" (A Killer Adversary for Quicksort, 1999)
// run against this libstdc++ std::sort: produces keys that drive introsort
// into its depth limit, so the heapsort fallback of the restatement is
// exercised by the tests.
namespace {
struct Adv {
  std::vector<int64_t> val;
  int64_t gas, nsolid = 0, candidate = 0;
  bool less(int64_t x, int64_t y) {
    if (val[x] == gas && val[y] == gas) {
      if (x == candidate) val[x] = nsolid++;
      else val[y] = nsolid++;
    }
    if (val[x] == gas) candidate = x;
    else if (val[y] == gas) candidate = y;
    return val[x] < val[y];
  }
};
}  // namespace

extern "C" void probe_antiqsort(int64_t n, int64_t* keys_out) {
  Adv adv;
  adv.gas = n;
  adv.val.assign(n, n);
  std::vector<int64_t> ptr(n);
  for (int64_t i = 0; i < n; ++i) ptr[i] = i;
  std::sort(ptr.begin(), ptr.end(), [&](int64_t a, int64_t b) { return adv.less(a, b); });
  for (int64_t i = 0; i < n; ++i) keys_out[i] = adv.val[i];
}
