"""Test-infrastructure oracle (CPU restatement of the reference path).

Never imported by the product package; see winograd_oracle.py's header.
"""
