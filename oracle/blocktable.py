"""CPU restatement of the device block tables (K8) -- TEST INFRASTRUCTURE ONLY.

Restates exactly what the executor does with a plan's KV ops
(paper_2402_01869_b200/csrc/exec/executor.cu apply_ops + k_misc.cu
block_update_kernel): per (request, logical block j = positions [16j,16j+16))
count resident positions; per phase, blocks whose count rose from zero are
allocations and blocks whose count fell to zero are frees (first-touch order);
the device pushes frees onto a LIFO stack of physical block ids, then pops one
per allocation.  The ledger semantics the ops come from are the reference's
(proj/src/memory.cpp:13-81); this restatement is what makes the device tables
checkable bit for bit.
"""
from __future__ import annotations

BLOCK = 16


class BlockTableOracle:
    def __init__(self, gpu_blocks: int):
        self.stack = list(range(gpu_blocks - 1, -1, -1))   # stack[top-1] is popped first
        self.count = {}     # (rid, lb) -> resident positions
        self.table = {}     # (rid, lb) -> physical block

    def _phase(self, ops, phase):
        touched, seen = [], set()

        def touch(rid, lo, hi, sign):
            b = lo // BLOCK
            while b * BLOCK < hi:
                key = (rid, b)
                if key not in seen:
                    seen.add(key)
                    touched.append((key, self.count.get(key, 0) > 0))
                a, e = max(lo, b * BLOCK), min(hi, (b + 1) * BLOCK)
                c = self.count.get(key, 0) + sign * (e - a)
                assert 0 <= c <= BLOCK, (key, c)
                self.count[key] = c
                b += 1

        for (rid, kind, ph, lo, hi) in ops:
            if ph != phase:
                continue
            if kind in (0, 2, 4):          # grow, swap-in, recompute
                touch(rid, lo, hi, +1)
            elif kind in (1, 3):           # swap-out, discard
                touch(rid, lo, hi, -1)
            elif kind == 5:                # release
                for key in [k for k in self.count if k[0] == rid and self.count[k] > 0]:
                    if key not in seen:
                        seen.add(key)
                        touched.append((key, True))
                    self.count[key] = 0
        frees = [k for k, was in touched if was and self.count.get(k, 0) == 0]
        allocs = [k for k, was in touched if not was and self.count.get(k, 0) > 0]
        for k in frees:
            self.stack.append(self.table.pop(k))
        for k in allocs:
            self.table[k] = self.stack.pop()
        for k in list(self.count):
            if self.count[k] == 0:
                del self.count[k]

    def apply(self, plan: dict) -> None:
        self._phase(plan["ops"], 0)
        self._phase(plan["ops"], 1)

    def table_of(self, rid: int, max_lb: int) -> list:
        return [self.table.get((rid, b), -1) for b in range(max_lb)]

    def free_blocks(self) -> int:
        return len(self.stack)
