// introsort.cuh -- device restatement of libstdc++ std::sort as scipy's
// csr_sort_indices uses it (std::pair<col, value>, comparator on col only).
//
// Why: scipy's coo->csr canonicalisation (graph.py:155-157 -> sum_duplicates)
// sorts every row with this UNSTABLE introsort whenever any row of the
// emitted COO has a column descent, then sums duplicate columns left to
// right.  fp64 addition is not associative, so a duplicate key with >= 3
// contributions of different 2/m values sums to the reference's bits only in
// the introsort's order.  The build pipeline
// (build.cu) sorts stably with a radix sort and calls this emulation only for
// the rows holding such order-sensitive keys.
//
// Published algorithm (bits/stl_algo.h, bits/stl_heap.h): median of
// (first+1, mid, last-1) moved to first, unguarded Hoare partition of
// [first+1, last), recurse right / loop left while the range exceeds 16,
// depth limit 2*floor(log2 n) -> heapsort, then a guarded insertion sort of
// the first 16 elements and an unguarded one of the rest.  The two halves
// produced by a partition are disjoint, so the device version walks them
// with an explicit stack instead of recursion; the final array is the same.
// Checked against the real std::sort by tests (oracle/stdsort_probe.cpp).
#pragma once

#include <stdint.h>

namespace gift {

struct KV {
  uint32_t k;
  uint32_t pad;
  double v;
};

__device__ __forceinline__ void kv_swap(KV* a, KV* b) {
  KV t = *a;
  *a = *b;
  *b = t;
}

__device__ inline void dev_move_median_to_first(KV* result, KV* a, KV* b, KV* c) {
  if (a->k < b->k) {
    if (b->k < c->k) kv_swap(result, b);
    else if (a->k < c->k) kv_swap(result, c);
    else kv_swap(result, a);
  } else if (a->k < c->k) {
    kv_swap(result, a);
  } else if (b->k < c->k) {
    kv_swap(result, c);
  } else {
    kv_swap(result, b);
  }
}

__device__ inline KV* dev_unguarded_partition(KV* first, KV* last, const KV* pivot) {
  const uint32_t pk = pivot->k;
  for (;;) {
    while (first->k < pk) ++first;
    --last;
    while (pk < last->k) --last;
    if (!(first < last)) return first;
    kv_swap(first, last);
    ++first;
  }
}

__device__ inline void dev_push_heap(KV* first, int64_t hole, int64_t top, KV value) {
  int64_t parent = (hole - 1) / 2;
  while (hole > top && first[parent].k < value.k) {
    first[hole] = first[parent];
    hole = parent;
    parent = (hole - 1) / 2;
  }
  first[hole] = value;
}

__device__ inline void dev_adjust_heap(KV* first, int64_t hole, int64_t len, KV value) {
  const int64_t top = hole;
  int64_t child = hole;
  while (child < (len - 1) / 2) {
    child = 2 * (child + 1);
    if (first[child].k < first[child - 1].k) child--;
    first[hole] = first[child];
    hole = child;
  }
  if ((len & 1) == 0 && child == (len - 2) / 2) {
    child = 2 * (child + 1);
    first[hole] = first[child - 1];
    hole = child - 1;
  }
  dev_push_heap(first, hole, top, value);
}

__device__ inline void dev_heap_sort(KV* first, KV* last) {
  const int64_t len = last - first;
  if (len >= 2) {
    int64_t parent = (len - 2) / 2;
    for (;;) {
      KV value = first[parent];
      dev_adjust_heap(first, parent, len, value);
      if (parent == 0) break;
      parent--;
    }
  }
  while (last - first > 1) {
    --last;
    KV value = *last;
    *last = *first;
    dev_adjust_heap(first, 0, last - first, value);
  }
}

__device__ inline void dev_unguarded_linear_insert(KV* last) {
  KV val = *last;
  KV* next = last - 1;
  while (val.k < next->k) {
    *last = *next;
    last = next;
    --next;
  }
  *last = val;
}

__device__ inline void dev_insertion_sort(KV* first, KV* last) {
  if (first == last) return;
  for (KV* i = first + 1; i != last; ++i) {
    if (i->k < first->k) {
      KV val = *i;
      for (KV* p = i; p != first; --p) *p = *(p - 1);
      *first = val;
    } else {
      dev_unguarded_linear_insert(i);
    }
  }
}

// std::sort(first, first + n) on KV by .k, single thread.
__device__ inline void dev_std_sort(KV* first, int64_t n) {
  if (n <= 0) return;
  KV* const end = first + n;
  struct Frame {
    KV* f;
    KV* l;
    int depth;
  };
  Frame stack[128];
  int sp = 0;
  stack[sp++] = {first, end, 2 * (63 - __clzll((unsigned long long)n))};
  while (sp > 0) {
    Frame fr = stack[--sp];
    KV* f = fr.f;
    KV* l = fr.l;
    int depth = fr.depth;
    while (l - f > 16) {
      if (depth == 0) {
        dev_heap_sort(f, l);
        break;
      }
      --depth;
      KV* mid = f + (l - f) / 2;
      dev_move_median_to_first(f, f + 1, mid, l - 1);
      KV* cut = dev_unguarded_partition(f + 1, l, f);
      stack[sp++] = {cut, l, depth};  // the recursive call on the right part
      l = cut;
    }
  }
  if (n > 16) {
    dev_insertion_sort(first, first + 16);
    for (KV* i = first + 16; i != end; ++i) dev_unguarded_linear_insert(i);
  } else {
    dev_insertion_sort(first, end);
  }
}

}  // namespace gift
