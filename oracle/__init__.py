"""CPU oracle for the BD K/V projection — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  The product package (paper_2510_01718_b200) never does.
"""
