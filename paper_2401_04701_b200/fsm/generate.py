"""Generate HiRace's constant-size per-word FSM table (build-time tool).

The paper's FSM "has 25 states and 1200 transitions" and "is encoded as a
flat array indexed by a concatenation of oState and the transition labels"
 but its states are never listed ("whose complete
specification will be made publicly available").  We
regenerate an equivalent machine from the design idea the paper states —
"we only track the hierarchical scope shared by the accessing threads"
 — as an abstract history relative to the last accessor
L, then Moore-minimise it.

Abstract history: for each access kind k in {R, W, A}, the set of CLASSES
present among the prior accesses of kind k, relative to L:

    F   another block than L
    BO  L's block, earlier block epoch (bc < L.bc)           - ordered
    WO  L's warp, same bc, earlier warp epoch (wc < L.wc)    - ordered
    S   L itself
    Wl  another lane of L's warp, same bc and wc             - unordered
    B   another warp of L's block, same bc                   - unordered

Transition for an access N with label (m, s, t) = (kind, sync status,
thread relation of N to L) — Algorithm 1's getTrans inputs:
  1. re-base every class to N (s = Bs orders all of L's block before N;
     s = Ws orders L's warp epoch; t = Global makes everything foreign ...),
  2. RACE iff some kind k conflicting with m has a class in {F, B, Wl}
     (unordered, distinct threads, at least one write; atomics
     per reading R1 of DESIGN.md),
  3. otherwise add S to kind m's set; N becomes the new L.
RACE is split into RACE_BLOCK / RACE_GRID (reading R4): GRID iff some prior
access was in another block than N (F present after re-basing); RACE_BLOCK
moves to RACE_GRID on any Global label.  INIT ignores the label
(SPEC.md:279).

Encoding:
    index = state << 6 | kind << 4 | sync << 2 | rel          (2048 bytes)
    kind  R=0 W=1 A=2      sync  Us=0 Ws=1 Bs=2      rel  Self=0 Warp=1 Block=2 Global=3
    INIT = 0 (the all-zero shadow word), RACE_BLOCK = 30, RACE_GRID = 31.
Infeasible labels (Bs with Global, Ws with Block/Global) are
never produced by hr__sync; their entries repeat the Us entry.  Sync index 3
(both bits: "bc and wc both differ") repeats the Bs entry (Bs dominates Ws,
SPEC.md:244), so a label computation may set the two bits independently
(bit 1 "block epoch differs", bit 0 "warp epoch differs") and let the table
resolve dominance and feasibility (hr__check_shared_row).
Per-state flag byte: bit0 race, bit1 label-insensitive closure (the stored
tid/clocks are dead: skip the write when the state is unchanged), bit2
block-only closure (only the stored block id is live: skip the write when the
state is unchanged and the relation is not Global).

Run ``python -m paper_2401_04701_b200.fsm.generate`` to regenerate
``csrc/fsm_table.inc``; tests/test_fsm.py checks the committed file is current.
"""
from __future__ import annotations

import os
from collections import deque
from typing import Dict, FrozenSet, Iterable, List, Optional, Sequence, Tuple

KINDS = ("R", "W", "A")
SYNCS = ("Us", "Ws", "Bs")
RELS = ("S", "W", "B", "G")
K_R, K_W, K_A = 0, 1, 2
S_US, S_WS, S_BS = 0, 1, 2
T_S, T_W, T_B, T_G = 0, 1, 2, 3

CLASSES = ("F", "BO", "WO", "S", "Wl", "B")
C_F, C_BO, C_WO, C_S, C_WL, C_B = (1 << i for i in range(6))
UNORDERED = C_F | C_B | C_WL

INIT_CODE = 0
RACE_BLOCK_CODE = 30
RACE_GRID_CODE = 31
N_CODES = 32

FLAG_RACE = 1
FLAG_INSENSITIVE = 2
FLAG_BLOCK_ONLY = 4

Hist = Tuple[int, int, int]            # class bitmask per kind
State = object                          # "INIT" | "RACE_BLOCK" | "RACE_GRID" | Hist


def feasible(s: int, t: int) -> bool:
    """Labels the label computation can produce."""
    if s == S_BS:
        return t != T_G
    if s == S_WS:
        return t in (T_S, T_W)
    return True


def all_labels(kinds=(K_R, K_W, K_A), syncs=(S_US, S_WS, S_BS), rels=(T_S, T_W, T_B, T_G)):
    return [(m, s, t) for m in kinds for s in syncs for t in rels if feasible(s, t)]


def conflict(m: int, k: int) -> bool:
    """At least one write; atomic-atomic never conflicts (reading R1)."""
    if m == K_R and k == K_R:
        return False
    if m == K_A and k == K_A:
        return False
    return True


def _rebase_mask(mask: int, s: int, t: int) -> int:
    out = mask & C_F                                   # F stays F (another block than L)
    rest = mask & ~C_F
    if not rest:
        return out
    if t == T_G:                                       # N in another block: all of L's block is foreign
        return out | C_F
    if s == S_BS:                                      # bc(N) > bc(L) >= bc of every entry of L's block
        return out | C_BO
    if s == S_WS:                                      # same warp, wc(N) > wc(L): L's warp epoch ordered
        if rest & (C_S | C_WL):
            out |= C_WO
        return out | (rest & (C_WO | C_B | C_BO))
    # s == Us
    if t == T_B:                                       # N: another warp of L's block, same bc
        if rest & (C_WO | C_S | C_WL | C_B):
            out |= C_B
        return out | (rest & C_BO)
    if t == T_W:                                       # N: another lane of L's warp, same epochs
        if rest & (C_S | C_WL):
            out |= C_WL
        return out | (rest & (C_WO | C_B | C_BO))
    return out | rest                                  # t == Self


def step(h: State, m: int, s: int, t: int, conflict_fn=None) -> State:
    """One FSM transition on the abstract history (module docstring).
    `conflict_fn` restricts the conflict relation (class projections)."""
    cf = conflict_fn or conflict
    if h == "RACE_GRID":
        return "RACE_GRID"
    if h == "RACE_BLOCK":
        return "RACE_GRID" if t == T_G else "RACE_BLOCK"
    if h == "INIT":
        hist = [0, 0, 0]
        hist[m] = C_S
        return tuple(hist)
    reb = [_rebase_mask(x, s, t) for x in h]           # type: ignore[union-attr]
    for k in range(3):
        if cf(m, k) and (reb[k] & UNORDERED):
            any_foreign = any(x & C_F for x in reb)
            return "RACE_GRID" if any_foreign else "RACE_BLOCK"
    reb[m] |= C_S
    return tuple(reb)


def hist_name(h: State) -> str:
    if isinstance(h, str):
        return h
    parts = []
    for k, mask in enumerate(h):
        if mask:
            cls = ",".join(c for i, c in enumerate(CLASSES) if mask & (1 << i))
            parts.append(f"{KINDS[k]}:{cls}")
    return "{" + " ".join(parts) + "}"


NAMED = {
    (C_S, 0, 0): "READ",
    (C_S | C_B, 0, 0): "BREAD",
    (C_S | C_F, 0, 0): "GREAD",
    (0, C_S, 0): "WRITE",
    (0, 0, C_S): "ATOMIC",
    (0, 0, C_S | C_B): "BATOMIC",
    (0, 0, C_S | C_F): "GATOMIC",
}


def closure(labels: Sequence[Tuple[int, int, int]], conflict_fn=None):
    """Reachable abstract histories from INIT under ``labels`` (BFS order)."""
    order: List[State] = ["INIT"]
    seen = {"INIT": 0}
    q = deque(["INIT"])
    while q:
        h = q.popleft()
        for (m, s, t) in labels:
            n = step(h, m, s, t, conflict_fn)
            if n not in seen:
                seen[n] = len(order)
                order.append(n)
                q.append(n)
    return order


def minimize(states: List[State], labels, output, conflict_fn=None) -> Dict[State, int]:
    """Moore partition refinement; returns state -> class id (ids in first-seen order)."""
    cls = {h: output(h) for h in states}
    while True:
        sig = {h: (cls[h],) + tuple(cls[step(h, m, s, t, conflict_fn)] for (m, s, t) in labels)
               for h in states}
        ids: Dict[tuple, int] = {}
        new = {}
        for h in states:
            new[h] = ids.setdefault(sig[h], len(ids))
        if len(set(new.values())) == len(set(cls.values())):
            return new
        cls = new


def _output_split(h: State):
    if h in ("INIT", "RACE_BLOCK", "RACE_GRID"):
        return h
    return "LIVE"


def _output_merged(h: State):
    if h in ("RACE_BLOCK", "RACE_GRID"):
        return "RACE"
    return "INIT" if h == "INIT" else "LIVE"


class Machine:
    """A minimised machine: codes, names, representatives, transition function."""

    def __init__(self, labels=None, split_race: bool = True, conflict_fn=None):
        self.labels = labels if labels is not None else all_labels()
        self.conflict_fn = conflict_fn
        states = closure(self.labels, conflict_fn)
        part = minimize(states, self.labels, _output_split if split_race else _output_merged, conflict_fn)
        # representative per class: first in BFS order (shortest history)
        rep: Dict[int, State] = {}
        for h in states:
            rep.setdefault(part[h], h)
        self.n_states = len(rep)
        self.part = part
        self.rep = rep
        # code assignment: INIT = 0, races = 30/31, live states 1.. in BFS order
        code: Dict[int, int] = {}
        nxt = 1
        for h in states:
            c = part[h]
            if c in code:
                continue
            if h == "INIT":
                code[c] = INIT_CODE
            elif h == "RACE_BLOCK":
                code[c] = RACE_BLOCK_CODE
            elif h == "RACE_GRID":
                code[c] = RACE_GRID_CODE if split_race else RACE_BLOCK_CODE
            else:
                code[c] = nxt
                nxt += 1
        if nxt > RACE_BLOCK_CODE:
            raise RuntimeError(f"{nxt} live states do not fit the 5-bit state field (PAPER.md:725)")
        self.code = code
        self.n_live = nxt - 1
        self.names = {}
        for c, h in rep.items():
            nm = NAMED.get(h) if isinstance(h, tuple) else h
            self.names[code[c]] = nm or hist_name(h)

    def code_of(self, h: State) -> int:
        return self.code[self.part[h]]

    def next_code(self, code: int, m: int, s: int, t: int) -> int:
        inv = {v: k for k, v in self.code.items()}
        h = self.rep[inv[code]]
        return self.code_of(step(h, m, s, t, self.conflict_fn))

    def codes(self) -> List[int]:
        return sorted(self.code.values())


def build_table(machine: Optional[Machine] = None):
    """The flat 2048-byte table and the 32-byte state-flag array."""
    mc = machine or Machine()
    table = bytearray(N_CODES * 64)
    inv = {v: k for k, v in mc.code.items()}
    for c in range(N_CODES):
        for kind in range(4):
            for s in range(4):
                for t in range(4):
                    idx = (c << 6) | (kind << 4) | (s << 2) | t
                    if c not in inv or kind == 3:
                        table[idx] = c
                        continue
                    ss = S_BS if s == 3 else s              # both bits set: Bs dominates Ws
                    ss = ss if feasible(ss, t) else S_US
                    table[idx] = mc.next_code(c, kind, ss, t)
    flags = bytearray(N_CODES)
    for c in mc.codes():
        if c in (RACE_BLOCK_CODE, RACE_GRID_CODE):
            flags[c] |= FLAG_RACE

    def insensitive(c):
        for m in range(3):
            vals = {table[(c << 6) | (m << 4) | (s << 2) | t] for s in range(3) for t in range(4) if feasible(s, t)}
            if len(vals) != 1:
                return False
        return True

    def block_only(c):
        for m in range(3):
            for g in (False, True):
                vals = {table[(c << 6) | (m << 4) | (s << 2) | t] for s in range(3) for t in range(4)
                        if feasible(s, t) and ((t == T_G) == g)}
                if len(vals) > 1:
                    return False
        return True

    def reach(c):
        seen, st = {c}, [c]
        while st:
            x = st.pop()
            for m in range(3):
                for s in range(3):
                    for t in range(4):
                        if feasible(s, t):
                            y = table[(x << 6) | (m << 4) | (s << 2) | t]
                            if y not in seen:
                                seen.add(y)
                                st.append(y)
        return seen

    for c in mc.codes():
        if c == INIT_CODE:
            continue
        r = reach(c)
        if all(insensitive(x) for x in r):
            flags[c] |= FLAG_INSENSITIVE
        if all(block_only(x) for x in r):
            flags[c] |= FLAG_BLOCK_ONLY
    return bytes(table), bytes(flags), mc


def render_inc(table: bytes, flags: bytes, mc: Machine) -> str:
    lines = ["/* GENERATED by paper_2401_04701_b200/fsm/generate.py — do not edit.",
             f" * {mc.n_states} states ({mc.n_live} live + INIT + RACE_BLOCK + RACE_GRID) over "
             f"{len(mc.labels)} feasible labels.",
             " * index = state<<6 | kind<<4 | sync<<2 | rel   (PAPER.md:741-743)"]
    for c in mc.codes():
        lines.append(f" *   {c:2d} {mc.names[c]}  flags={flags[c]}")
    lines.append(" */")
    lines.append("#define HR_FSM_N_STATES %d" % mc.n_states)
    lines.append("static const unsigned char hr_fsm_table_init[2048] = {")
    for c in range(N_CODES):
        row = table[c * 64:(c + 1) * 64]
        lines.append("  " + ",".join(str(x) for x in row) + ",")
    lines.append("};")
    lines.append("static const unsigned char hr_fsm_flags_init[32] = {")
    lines.append("  " + ",".join(str(x) for x in flags))
    lines.append("};")
    return "\n".join(lines) + "\n"


# ---- per-pair race classes ---------------------------------
# Class c is a kind pair; its projection sees only the accesses of those kinds
# and calls a pair a conflict only when it is of class c.  A projection enters
# RACE iff the word has a race pair of class c (verified against the oracle's
# classes in tests/test_fsm.py).  Encoding as the main table; RACE = 30.
CLASSES_PAIRS = (("WW", (K_W,), lambda m, k: m == K_W and k == K_W),
                 ("RW", (K_R, K_W), lambda m, k: {m, k} == {K_R, K_W}),
                 ("AW", (K_A, K_W), lambda m, k: {m, k} == {K_A, K_W}),
                 ("AR", (K_A, K_R), lambda m, k: {m, k} == {K_A, K_R}))


def class_machines():
    out = []
    for name, kinds, cf in CLASSES_PAIRS:
        mc = Machine(labels=all_labels(kinds=kinds), split_race=False, conflict_fn=cf)
        table = bytearray(N_CODES * 64)
        inv = {v: k for k, v in mc.code.items()}
        for c in range(N_CODES):
            for kind in range(4):
                for sy in range(4):
                    for t in range(4):
                        idx = (c << 6) | (kind << 4) | (sy << 2) | t
                        if c not in inv or kind not in kinds:
                            table[idx] = c
                            continue
                        ss = sy if (sy < 3 and feasible(sy, t)) else S_US
                        table[idx] = mc.next_code(c, kind, ss, t)
        out.append((name, kinds, bytes(table), mc))
    return out


def render_classes_inc(machines) -> str:
    lines = ["/* GENERATED by paper_2401_04701_b200/fsm/generate.py — do not edit.",
             " * Race-class projections (SURVEY §8(f)-3): table c sees kinds of class c",
             " * only; RACE (code 30) iff the word has a race pair of that class."]
    for name, kinds, _, mc in machines:
        lines.append(f" *   {name}: kinds {'/'.join(KINDS[k] for k in kinds)}, {mc.n_states} states")
    lines.append(" */")
    mask = [sum(1 << k for k in kinds) for _, kinds, _, _ in machines]
    lines.append("static const unsigned char hr_class_kinds_init[4] = {" + ",".join(str(x) for x in mask) + "};")
    lines.append("static const unsigned char hr_class_tables_init[4][2048] = {")
    for name, _, table, _ in machines:
        lines.append("  { /* " + name + " */")
        for c in range(N_CODES):
            lines.append("    " + ",".join(str(x) for x in table[c * 64:(c + 1) * 64]) + ",")
        lines.append("  },")
    lines.append("};")
    return "\n".join(lines) + "\n"


CLASSES_INC_PATH = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "csrc",
                                "fsm_classes.inc")

INC_PATH = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "csrc", "fsm_table.inc")


def main() -> None:
    table, flags, mc = build_table()
    with open(INC_PATH, "w") as f:
        f.write(render_inc(table, flags, mc))
    print(f"wrote {INC_PATH}: {mc.n_states} states")
    cms = class_machines()
    with open(CLASSES_INC_PATH, "w") as f:
        f.write(render_classes_inc(cms))
    print(f"wrote {CLASSES_INC_PATH}: " + ", ".join(f"{n} {m.n_states} states" for n, _, _, m in cms))
    for c in mc.codes():
        print(f"  {c:2d} {mc.names[c]:32s} flags={flags[c]}")


if __name__ == "__main__":
    main()
