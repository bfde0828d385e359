"""The reference's per-window sort API (pkg/src/irdenoise/sorting.py), on the CPU.

`run_filter` never calls this module: the kernels select medians with exact
selection networks and bitwise rank selection (csrc/select_nets.cuh,
csrc/fnr_large.cuh), which give the same value as any exact sort. It exists so that
code written against the reference's public surface (`irdenoise.__init__:44`:
`SortCounters`, `median_of`, `sort_values`) keeps working, with the same results
AND the same instrumentation counters:

* `sort_values` (sorting.py:35-48): a sorted copy; introsort when n > 16 — median-of-3
  Hoare partitions, heapsort once the depth budget 2*floor(log2 n) is spent
  (counted in `depth_switches`), partitions of <= 16 elements left for one final
  insertion pass over the whole buffer (sorting.py:59-161);
* `median_of` (sorting.py:51-56): element (n-1)//2 of one counted sort, odd n only;
* `SortCounters` (sorting.py:19-32): sorts performed, element comparisons, depth switches.

The recursion of the reference's quicksort loop is replaced by an explicit work list
of (lo, hi, depth) ranges; ranges are disjoint, so the visiting order changes neither
the result nor any counter.
"""

from __future__ import annotations

INSERTION_CUTOFF = 16  # sorting.py:16


class SortCounters:
    """Monotone tallies of the sort instrumentation (sorting.py:19-32)."""

    __slots__ = ("sorts_performed", "comparisons", "depth_switches")

    def __init__(self) -> None:
        self.sorts_performed = 0
        self.comparisons = 0
        self.depth_switches = 0

    def merge(self, other: "SortCounters") -> None:
        self.sorts_performed += other.sorts_performed
        self.comparisons += other.comparisons
        self.depth_switches += other.depth_switches


class _Introsort:
    """One instrumented sort of a private buffer; `comps` accumulates comparisons."""

    def __init__(self, buf: list) -> None:
        self.a = buf
        self.comps = 0
        self.switches = 0

    def run(self) -> None:
        a = self.a
        n = len(a)
        if n > INSERTION_CUTOFF:
            work = [(0, n, 2 * (n.bit_length() - 1))]
            while work:
                lo, hi, budget = work.pop()
                while hi - lo > INSERTION_CUTOFF:
                    if budget == 0:
                        self.switches += 1
                        self.heapsort(lo, hi)
                        break
                    budget -= 1
                    cut = self.hoare(lo, hi)
                    work.append((cut, hi, budget))
                    hi = cut
        self.insertion(0, n)

    def hoare(self, lo: int, hi: int) -> int:
        """Median-of-3 pivot into a[mid], then Hoare scans; returns the split point."""
        a = self.a
        mid, last = (lo + hi) // 2, hi - 1
        if a[mid] < a[lo]:
            a[lo], a[mid] = a[mid], a[lo]
        self.comps += 2
        if a[last] < a[mid]:
            a[mid], a[last] = a[last], a[mid]
            self.comps += 1
            if a[mid] < a[lo]:
                a[lo], a[mid] = a[mid], a[lo]
        pivot = a[mid]
        i, j = lo, last
        while True:
            i += 1
            while a[i] < pivot:
                i += 1
                self.comps += 1
            j -= 1
            while a[j] > pivot:
                j -= 1
                self.comps += 1
            self.comps += 2  # the two failed scan tests
            if i >= j:
                return j + 1
            a[i], a[j] = a[j], a[i]

    def heapsort(self, lo: int, hi: int) -> None:
        a, n = self.a, hi - lo

        def sift(root: int, end: int) -> None:
            while True:
                child = 2 * root + 1
                if child >= end:
                    return
                if child + 1 < end:
                    self.comps += 1
                    if a[lo + child] < a[lo + child + 1]:
                        child += 1
                self.comps += 1
                if not a[lo + root] < a[lo + child]:
                    return
                a[lo + root], a[lo + child] = a[lo + child], a[lo + root]
                root = child

        for root in range(n // 2 - 1, -1, -1):
            sift(root, n)
        for end in range(n - 1, 0, -1):
            a[lo], a[lo + end] = a[lo + end], a[lo]
            sift(0, end)

    def insertion(self, lo: int, hi: int) -> None:
        a = self.a
        for i in range(lo + 1, hi):
            v = a[i]
            j = i - 1
            while j >= lo:
                self.comps += 1
                if not a[j] > v:
                    break
                a[j + 1] = a[j]
                j -= 1
            a[j + 1] = v


def sort_values(values, counters: SortCounters) -> list[int]:
    """A new non-decreasing list of the values; counts one sort (sorting.py:35-48).

    Raises ValueError on empty input."""
    s = _Introsort(list(values))
    if not s.a:
        raise ValueError("cannot sort an empty sequence")
    s.run()
    counters.comparisons += s.comps
    counters.depth_switches += s.switches
    counters.sorts_performed += 1
    return s.a


def median_of(values, counters: SortCounters) -> int:
    """Median of an odd-length sequence via one counted sort (sorting.py:51-56)."""
    n = len(values)
    if n % 2 == 0:
        raise ValueError(f"median needs an odd-length sequence, got length {n}")
    return sort_values(values, counters)[(n - 1) // 2]
