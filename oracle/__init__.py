"""Plain CPU oracle of the PIC step -- TEST INFRASTRUCTURE ONLY (see pic_oracle.h)."""
