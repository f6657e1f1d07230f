"""ORACLE — test infrastructure only (see oracle/oracle.py).  Never imported by
the product package paper_2302_06173_b200."""
