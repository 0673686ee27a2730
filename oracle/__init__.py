"""CPU oracle -- TEST INFRASTRUCTURE ONLY (see lg_oracle.py).  Never imported by the product."""
