"""Benchmark / test input generation (libscene.so): not part of the product."""
