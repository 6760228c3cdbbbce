"""ORACLE / TEST INFRASTRUCTURE (see oracle/oracle.py). Never imported by the product."""
