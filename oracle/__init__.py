"""Test infrastructure: the CPU oracle and the recipe that builds the real
reference into oracle/_ref.  Not part of the product."""
