"""The oracle's pins kill every listed mutation of the oracle (tools/mutation_check.py).

A pin that no plausible misreading of the paper's method can pass is what makes the
oracle's parity claims mean something (SURVEY.md §8(c) "Pins"): each
mutation of oracle/oracle.c — the AV clamp and sign, the limiter, the sound speed, the
softening form, the predicate and a dozen more — must make at least one CPU pin fail.
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "tools"))


def test_every_oracle_mutation_is_killed():
    import mutation_check

    assert mutation_check.main([]) == 0
