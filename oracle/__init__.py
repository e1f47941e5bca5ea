"""CPU checkers for the COVAP path — TEST INFRASTRUCTURE ONLY (see oracle.py)."""
