"""Bench / test tooling (synthetic inputs, microbenchmarks); not the product."""
