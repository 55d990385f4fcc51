"""TEST INFRASTRUCTURE — CPU oracle for the PbP-QLP path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package.  The product package
(paper_2103_07245_b200) never imports it; it is the checker, not the path.
"""
