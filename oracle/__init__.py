"""Test infrastructure only: the CPU oracle for parity checks and the CPU baseline timing.

Never imported by the product package (paper_2309_00628_b200).
"""
