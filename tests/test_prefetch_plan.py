"""``plan_early_fetches``: where ADAM's fetches are issued ahead of the ledger
(host logic of the payload executor; no GPU).  Properties: every placed fetch
fits, together with every fetch placed at or before its event, under the
capacity minus the margin at every later moment up to the one before ADAM
(ADAM's own usage already counts them); placement is as
early as that allows; the walk's order is kept; nothing lands after the last
event."""

import random

from paper_2108_05818_b200.payload import plan_early_fetches


def _check(fetches, used, cap, margin, adam, last, out):
    placed = [(e, cid) for e, ids in out.items() for cid in ids]
    order = [cid for _, cid in sorted(placed, key=lambda x: (x[0], [c for c, _ in fetches].index(x[1])))]
    assert order == [cid for cid, _ in fetches][:len(order)]  # a prefix, in walk order
    size = dict(fetches)
    peak = {}
    for m, b in used:
        peak[m] = max(peak.get(m, 0), b)
    for e, cid in placed:
        assert e <= last
        held = sum(size[c] for f, c in placed if f <= e or order.index(c) <= order.index(cid))
        for m in range(2 * e, 2 * adam + 1):  # up to the moment before ADAM
            assert peak.get(m, 0) + held <= cap - margin, (e, cid, m)
        # not placeable one event earlier
        if e > min(peak) // 2:
            held_before = sum(size[c] for c in order[:order.index(cid) + 1])
            assert any(peak.get(m, 0) + held_before > cap - margin
                       for m in range(2 * (e - 1), 2 * adam + 1))


def test_known_answer():
    # backward frees 10 per event from 100 down to 20; ADAM at event 9
    used = [(2 * e, 100 - 10 * e) for e in range(10)] + [(2 * e + 1, 100 - 10 * e)
                                                        for e in range(10)]
    fetches = [(1, 20), (2, 20), (3, 20)]
    out = plan_early_fetches(fetches, used, capacity=110, margin=0, adam_index=9, last_event=7)
    # room capacity - usage: e=0 10, e=1 20, e=2 30, e=3 40, e=4 50, e=5 60 ...
    assert out == {1: [1], 3: [2], 5: [3]}
    _check(fetches, used, 110, 0, 9, 7, out)


def test_no_room_before_last_event_leaves_the_rest():
    used = [(m, 100) for m in range(20)]
    out = plan_early_fetches([(1, 5), (2, 5)], used, capacity=108, margin=0, adam_index=9,
                             last_event=7)
    assert out == {0: [1]}  # the second would exceed 108 anywhere: left to the normal prefetch


def test_random_schedules():
    r = random.Random(7)
    for _ in range(300):
        adam = r.randint(3, 40)
        base = r.randint(50, 200)
        used = []
        level = base
        for e in range(adam + 1):
            level = max(0, level + r.randint(-30, 20))
            used.append((2 * e, level))
            used.append((2 * e + 1, level + r.randint(0, 10)))
        cap = max(b for _, b in used) + r.randint(0, 100)
        margin = r.randint(0, 10)
        fetches = [(i, r.randint(1, 40)) for i in range(r.randint(1, 12))]
        last = adam - r.randint(1, 2)
        out = plan_early_fetches(fetches, used, cap, margin, adam, last)
        _check(fetches, used, cap, margin, adam, last, out)
