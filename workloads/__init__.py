"""Synthetic bench/test workloads (builder-defined): the design-space
catalogue and the seeded tuning tasks. Pure Python; imports nothing from the product."""
