"""Host-side logic of the path that needs no GPU."""
from paper_2506_17551_b200.parsim import StalenessTracker


def test_staleness_tracker_invariants():
    """test_strategies.cpp:86-95 (parsim/strategies.hpp:65-77)."""
    tr = StalenessTracker(3)
    assert tr.workers() == 3
    assert tr.staleness(0) == 0
    tr.on_global_update()
    tr.on_global_update()
    assert tr.staleness(1) == 2
    tr.on_pull(1)
    assert tr.staleness(1) == 0
    assert tr.staleness(2) == 2


def test_staleness_tracker_reproduces_trainer_tau_pattern():
    """The trainer's async branch (trainer.hpp:244-255) pulls one snapshot per
    group of s+1 workers: tracking pulls and updates with the tracker gives
    tau_p = min(updates, p mod (s+1)) for every worker of every round."""
    for s in (1, 2, 3):
        P = 8
        tr = StalenessTracker(P)
        updates = 0
        for _round in range(3):
            for p in range(P):
                if p % (s + 1) == 0:      # the group's snapshot is taken here
                    for q in range(p, min(P, p + s + 1)):
                        tr.on_pull(q)
                assert tr.staleness(p) == min(updates, p % (s + 1))
                tr.on_global_update()
                updates += 1
