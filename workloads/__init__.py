"""Seeded synthetic inputs shared by the tests, the bench and smoke().

This package holds NONE of the method's arithmetic: it only draws random numbers
(the counter-based hash of SURVEY.md 8(d)) and writes problem statements in the
term format of include/hobo.h (coefficient x product of affine factors).  Both the
oracle (oracle/) and the product (paper_2407_19987_b200/) consume what it emits;
it imports neither.
"""
from .gen import *  # noqa: F401,F403
